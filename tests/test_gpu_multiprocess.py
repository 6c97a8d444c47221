"""The consensus round across two PROCESSES with libbsgpu's real kernels
(pack, unpack, residual and diagnostic reductions of csrc/consensus.cu): two
contexts on the one GPU of this box, one per process, their all-reduces
joined by a torch.distributed gloo group through the host communicator
(bsg_comm_init_host) -- the multi-rank protocol of SURVEY §8(e) with the
product code on both ranks, checked against the oracle's consensus_average /
dual_update / residuals / max_disagreement (admm.cpp:56-243)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import _oracle as orc
from gpu_helpers import gpu
from refcases import HostCloud
from test_gpu_train import make_blocks_for_consensus, rows_of

pytestmark = gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("relax,fd", [(False, 3), (True, 3), (True, 12)])
def test_two_process_round_matches_oracle(tmp_path, relax, fd):
    port = free_port()
    procs, outs = [], []
    for rank in range(2):
        out = tmp_path / f"rank{rank}.json"
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   RELAX="1" if relax else "0", FD=str(fd), OUT=str(out))
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "mp_consensus_worker.py")], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
        outs.append(out)
    for p in procs:
        log, _ = p.communicate(timeout=240)
        assert p.returncode == 0, log
    got = [json.load(open(o)) for o in outs]
    a, b, shared, zprev = make_blocks_for_consensus(fd=fd)
    alpha = 1.6
    sa = orc.slice_by_ids(a.oracle(), shared)
    sb = orc.slice_by_ids(b.oracle(), shared)
    z, flipped = orc.consensus_average([(0, sa), (1, sb)], relax, zprev.oracle(), alpha)
    zr = rows_of(HostCloud.from_oracle(z))
    p, d = orc.residuals([(0, sa), (1, sb)], z, zprev.oracle(), orc.Penalties())
    for r, (g, hc) in enumerate(zip(got, (a, b))):
        np.testing.assert_allclose(np.array(g["z"]), zr, rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(np.array(g["anchor"]), zr, rtol=1e-6, atol=1e-6)
        x = rows_of(HostCloud.from_oracle(orc.slice_by_ids(hc.oracle(), shared)))
        xh = alpha * x + (1 - alpha) * rows_of(zprev) if relax else x
        want_u = xh - zr
        for k, gid in enumerate(shared):
            if gid in flipped:
                want_u[k] = 0
        np.testing.assert_allclose(np.array(g["duals"]), want_u, rtol=1e-5, atol=2e-6)
        res = g["res"]
        assert res["flipped"] == len(flipped) == 1
        assert res["primal"] == pytest.approx(p, rel=1e-5)
        assert res["dual"] == pytest.approx(d, rel=1e-4)
        assert res["max_disagreement"] == pytest.approx(orc.max_disagreement([(0, sa), (1, sb)]), rel=1e-5)
        ops = [c[2] for c in g["calls"]]
        assert "sum" in ops and "max" in ops  # the diagnostics reductions ran through the hook too
    # both ranks hold bit-identical replicated results
    assert got[0]["z"] == got[1]["z"] and got[0]["res"]["primal"] == got[1]["res"]["primal"]
