"""Multi-rank host logic on CPU (gloo, world_size 2): every rank derives the
same block plan with the native planner, the per-rank slot tables cover the
global slot table with the right owner counts and one first owner per slot,
and the consensus protocol the device runs over NCCL (q-reference
pre-reduction, sum of relaxed sign-aligned contributions + flip flags, then a
3-double reduction of the residual / flip partials, each slot's dual residual
counted by its lowest owner) reproduces the reference's consensus_average /
dual_update / residuals when the sums are done by torch.distributed, with
identical residuals and penalty decisions on every rank. The pack/unpack here
is a numpy restatement of csrc/consensus.cu for the protocol check only."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import _oracle as orc
from paper_2405_13943_b200 import api
from paper_2405_13943_b200.scene import aerial_scene
from refcases import HostCloud

ALPHA = 1.6


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def rows(hc):
    return np.concatenate([hc.pos, hc.rot, hc.ls, hc.feat, hc.op[:, None]], 1)


def scene():
    cloud, cams = aerial_scene(3000, 64, 48, 8, 20.0, seed=9)
    hc = HostCloud(cloud["ids"], cloud["pos"], cloud["rot"], cloud["ls"], cloud["feat"], cloud["op"])
    # per-block "trained" copies: perturb each block's rows differently, flip some quaternions
    return hc, np.array([c.center() for c in cams])


def block_params(hc, ids, rank):
    g = np.random.default_rng(100 + rank)
    sel = ids.astype(np.int64)
    b = HostCloud(hc.ids[sel], hc.pos[sel] + 0.01 * g.normal(size=(len(sel), 3)), hc.rot[sel].copy(),
                  hc.ls[sel] + 0.01 * g.normal(size=(len(sel), 3)), hc.feat[sel], hc.op[sel] + 0.1 * rank)
    if rank == 1:
        b.rot[::7] *= -1.0  # antipodal copies must be sign-aligned to the first owner
    return b.narrowed()


def worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hc, centers = scene()
    plan = api.Plan(hc.ids, hc.pos, centers, world, 1.4)
    sids, owners, first_owner = plan.shared()
    ids, _ = plan.block(rank)
    r_rows, slots, first = plan.block_shared(rank)
    mine = block_params(hc, ids, rank)
    S, D = len(sids), 14
    zprev = rows(hc)[sids.astype(np.int64)].astype(np.float32)
    x = rows(mine)[r_rows].astype(np.float32)
    # reduction 1: q of the lowest owner
    qref = np.zeros((S, 4), np.float32)
    qref[slots[first == 1]] = x[first == 1, 3:7]
    t = torch.from_numpy(qref)
    dist.all_reduce(t)
    qref = t.numpy()
    # reduction 2: relaxed, sign-aligned contributions + flip flags
    xq = x.copy()
    dot = (xq[:, 3:7] * qref[slots]).sum(1)
    flip = (first == 0) & (dot < 0)
    xq[flip, 3:7] *= -1
    contrib = ALPHA * xq + (1 - ALPHA) * zprev[slots]
    pack = np.zeros((S, D + 1), np.float32)
    pack[slots, :D] = contrib
    pack[slots, D] = flip
    t = torch.from_numpy(pack)
    dist.all_reduce(t)
    pack = t.numpy()
    z = pack[:, :D] / owners[:, None]
    flipped = np.nonzero(pack[:, D] > 0)[0]
    # dual update (no sign flip on x_hat), resets of flipped slots
    xh = ALPHA * x + (1 - ALPHA) * zprev[slots]
    u = xh - z[slots]
    u[np.isin(slots, flipped)] = 0
    # residual partials -> one 3-double all-reduce (csrc/consensus.cu unpack_own_kernel):
    # primal^2 over own rows; dual^2 and flips over the slots this rank leads
    rho = api.penalties()
    rho_c = np.array([rho.rho_p] * 3 + [rho.rho_q] * 4 + [rho.rho_s] * 3 + [rho.rho_f] * 3 + [rho.rho_o], np.float64)
    lead = first == 1
    zf = z[slots].astype(np.float64)
    p2 = float(((x.astype(np.float64) - zf) ** 2).sum())
    d2 = float(((rho_c * (zf[lead] - zprev[slots][lead].astype(np.float64))) ** 2).sum())
    fl = float((pack[slots, D] > 0)[lead].sum())
    scal = torch.tensor([p2, d2, fl], dtype=torch.float64)
    dist.all_reduce(scal)
    primal, dual = float(np.sqrt(scal[0].item())), float(np.sqrt(scal[1].item()))
    # adapt_penalties (admm.cpp:200-217) on the reduced, rank-identical values
    f = 2.0 if primal > 10.0 * dual else (0.5 if dual > 10.0 * primal else 1.0)
    out_q.put((rank, dict(ids=ids, slots=slots, first=first, sids=sids, owners=owners, z=z, flipped=flipped,
                          u=u, primal=primal, dual=dual, flips=int(scal[2].item()), rho_factor=f, x=rows(mine),
                          zprev=zprev)))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_consensus_protocol_matches_reference():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0, r1 = res[0], res[1]
    # identical plans on every rank
    assert np.array_equal(r0["sids"], r1["sids"]) and np.array_equal(r0["owners"], r1["owners"])
    S = len(r0["sids"])
    assert S > 0
    cover = np.zeros(S, int)
    firsts = np.zeros(S, int)
    for r in (r0, r1):
        cover[r["slots"]] += 1
        firsts[r["slots"]] += r["first"]
    assert np.array_equal(cover, r0["owners"]) and np.all(firsts == 1)
    # reference consensus over the same shared slices
    hc, _ = scene()
    locs = []
    for b, r in ((0, r0), (1, r1)):
        ids = r["ids"]
        blk = HostCloud(ids, r["x"][:, 0:3], r["x"][:, 3:7], r["x"][:, 7:10], r["x"][:, 10:13], r["x"][:, 13])
        locs.append((b, orc.slice_by_ids(blk.oracle(), list(r["sids"]))))
    zp = HostCloud(r0["sids"], r0["zprev"][:, 0:3], r0["zprev"][:, 3:7], r0["zprev"][:, 7:10], r0["zprev"][:, 10:13],
                   r0["zprev"][:, 13])
    z, flipped = orc.consensus_average(locs, True, zp.oracle(), ALPHA)
    zr = rows(HostCloud.from_oracle(z))
    np.testing.assert_allclose(r0["z"], zr, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(r1["z"], zr, rtol=1e-5, atol=1e-5)
    assert sorted(r0["sids"][r0["flipped"]].tolist()) == sorted(flipped)
    primal, dual = orc.residuals(locs, z, zp.oracle(), orc.Penalties())
    assert r0["primal"] == pytest.approx(primal, rel=1e-4)
    assert r0["dual"] == pytest.approx(dual, rel=1e-4)
    # every rank holds bit-identical residuals, flip count and penalty decision
    assert (r0["primal"], r0["dual"], r0["flips"], r0["rho_factor"]) == (r1["primal"], r1["dual"], r1["flips"],
                                                                         r1["rho_factor"])
    assert r0["flips"] == len(flipped)
    for b, r in ((0, r0), (1, r1)):
        xs = rows(HostCloud.from_oracle(orc.slice_by_ids(locs[b][1], list(r0["sids"][r["slots"]]))))
        u = orc.dual_update(orc.zero_bundle(list(r0["sids"][r["slots"]]), 3),
                            orc.slice_by_ids(HostCloud(r0["sids"][r["slots"]], *(np.split(
                                (ALPHA * xs + (1 - ALPHA) * r0["zprev"][r["slots"]]), [3, 7, 10, 13], 1))).oracle(),
                                             list(r0["sids"][r["slots"]])), z)
        ur = rows(HostCloud.from_oracle(u))
        ur[np.isin(r["slots"], r0["flipped"])] = 0
        np.testing.assert_allclose(r["u"], ur, rtol=1e-4, atol=1e-5)
