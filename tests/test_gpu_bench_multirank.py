"""bench.py's N > 1 flow (torchrun, one block per rank, asynchronous rounds,
max-over-ranks timing, the consensus keys of the JSON line) run on this
box's single GPU: two ranks share it, so their rounds go through the host
communicator over a gloo group instead of NCCL (the 8-GPU layout uses one
NCCL rank per GPU; the kernels and the protocol are the same)."""
import json
import os
import socket
import subprocess
import sys

from gpu_helpers import gpu

pytestmark = gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_on_one_gpu():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "cfg2",
           "--gaussians", "400000", "--steps", "60", "--warmup", "3", "--interval", "10", "--no-also", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["block_steps_per_s"] == 2 * d["value"]
    assert d["config"]["blocks"] == 2 and d["config"]["shared_ids"] > 0
    c = d["consensus"]
    assert c["round_ms_device"] > 0 and 0 < c["comm_fraction"] < 1
    assert d["consensus_ms_per_iter"] > 0 and "exposed_fraction" in c
