"""The device invariant checks (BSG_DASSERT, csrc/bsg_internal.cuh) over a run
of every entry point (tests/checked_workload.py) with the checked library
lib/libbsgpu_checked.so: a tile cursor leaving its range, an entry index past
the staged batch, a sort larger than its shared memory, a gradient slot or
anchor index out of bounds traps the kernel and fails the run. (This pool has
compute-sanitizer closed; these are the library's own bounds checks, next to
the oracle comparisons of every other test.)"""
import os
import subprocess
import sys

from gpu_helpers import gpu
from paper_2405_13943_b200 import api

pytestmark = gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_checked_build_runs_clean():
    lib = os.path.join(os.path.dirname(api.LIB_PATH), "libbsgpu_checked.so")
    assert os.path.exists(lib), "run __graft_entry__.build()"
    env = dict(os.environ, BSG_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(HERE, "checked_workload.py")], capture_output=True, text=True,
                       timeout=900, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "BSG_DASSERT" not in out and "checked workload done" in out


def test_checked_build_traps_a_violation():
    """The checks are live: the checked library's probe kernel fails its check
    on purpose and the entry point reports the trap (in a throwaway process:
    a trap poisons the CUDA context); the normal library has none."""
    lib = os.path.join(os.path.dirname(api.LIB_PATH), "libbsgpu_checked.so")
    code = ("import sys; sys.path.insert(0, %r); from paper_2405_13943_b200 import api; L = api.load_library(); "
            "print('checked', L.bsg_checked_build(), 'probe', L.bsg_checked_probe(0))" % os.path.dirname(HERE))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, BSG_LIB=lib))
    assert "checked 1 probe %d" % api.BSG_ERR_CUDA in r.stdout, r.stdout + r.stderr
    assert "BSG_DASSERT failed" in r.stdout + r.stderr
    lib = api.load_library()
    assert lib.bsg_checked_build() == 0
