"""The master round's ownership bookkeeping (runtime.cpp:490-518) on the
device (bsg_owners_*) against the oracle's restatement, with
identical removed / new id lists: reset, unshared and dead ids and the shared
set after each round must be identical (integer contract)."""
import numpy as np
import pytest

import _oracle as orc
from gpu_helpers import gpu
from paper_2405_13943_b200 import api

pytestmark = gpu


def device_round(table, S, removed):
    """One round through the device table -> (reset, unshared, dead, shared_now)."""
    slots, cls, masks, found = table.remove(removed)
    S = np.asarray(S, np.uint64)
    reset = sorted(int(S[s]) for s, c in zip(slots, cls) if c == 1)
    unshared = sorted(int(S[s]) for s, c in zip(slots, cls) if c == 2)
    dead = [int(S[s]) for s, c in zip(slots, cls) if c == 3]
    flat = [int(i) for r in removed for i in r]
    dead += [i for i, f in zip(flat, found) if not f]  # single-owner ids: removal kills them
    ids, _ = table.table()
    return reset, unshared, sorted(set(dead)), [int(i) for i in ids]


@pytest.mark.parametrize("blocks,n,seed", [(2, 2000, 1), (4, 20000, 2), (8, 50000, 3), (32, 5000, 4)])
def test_owner_table_matches_master_bookkeeping(blocks, n, seed):
    g = np.random.default_rng(seed)
    owners = {}
    for i in range(n):
        k = int(g.integers(1, min(blocks, 4) + 1))
        owners[i * 3 + 1] = sorted(int(b) for b in g.choice(blocks, size=k, replace=False))
    next_id = [(b << 48) + (n * 3 + 10 if b == 0 else 0) for b in range(blocks)]  # IdAllocator::for_block
    shared = sorted(i for i, o in owners.items() if len(o) >= 2)
    masks = [sum(1 << b for b in owners[i]) for i in shared]
    table = api.OwnerTable(shared, masks, blocks)
    S = shared
    for rnd in range(3):
        removed = [[] for _ in range(blocks)]
        for i, o in owners.items():
            for b in o:
                if g.random() < 0.15:
                    removed[b].append(i)
        added = []
        for b in range(blocks):
            k = int(g.integers(0, 20))
            added.append(list(range(next_id[b], next_id[b] + k)))
            next_id[b] += k
        removed = [sorted(r) for r in removed]
        want = orc.master_ownership_round(owners, removed, added)
        got = device_round(table, S, removed)
        assert got[0] == list(want["reset"]), rnd
        assert got[1] == list(want["unshared"]), rnd
        assert got[2] == list(want["dead"]), rnd
        assert got[3] == list(want["shared_now"]), rnd
        assert (len(want["reset"]) > 0 or blocks == 2) and len(want["unshared"]) > 0 and len(want["dead"]) > 0
        owners = {int(k): list(v) for k, v in want["owners"].items()}
        S = got[3]
        # the device masks are the oracle's owner lists of the shared ids
        ids, m = table.table()
        for i, mk in zip(ids, m):
            assert mk == sum(1 << b for b in owners[int(i)])
    table.close()


def test_owner_table_rejects_bad_rows():
    with pytest.raises(api.InvalidArgument):
        api.OwnerTable([5, 3], [3, 3], 2)  # not ascending
    with pytest.raises(api.InvalidArgument):
        api.OwnerTable([1, 2], [3, 1], 2)  # a single-owner row
