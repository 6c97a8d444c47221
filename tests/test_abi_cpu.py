"""CPU-side checks of the C-ABI boundary: the shared library loads, exports
every function include/bsgpu.h declares, and fails loudly (no CPU fallback)
when no B200 is present. No compute calls."""
import ctypes
import os
import re

import pytest

from paper_2405_13943_b200 import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bsgpu.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bsg_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    names = declared_functions()
    assert len(names) >= 30
    assert names == sorted(n for n, _, _ in api.SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(api.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", api.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_abi_version_and_defaults():
    lib = api.load_library()
    assert lib.bsg_abi_version() == 1
    r = api.render_config()
    assert (r.near_plane, r.dilation, r.alpha_clamp, r.transmittance_stop, r.sigma_extent, r.lambda_) == (
        0.01, 0.3, 0.99, 1e-4, 3.0, 0.2)  # renderer.hpp:13-21
    t = api.trainer_config()
    assert (t.lr_position, t.lr_position_decay, t.lr_rotation, t.lr_log_scale, t.lr_features, t.lr_opacity) == (
        1.6e-4, 0.01, 1e-3, 5e-3, 2.5e-3, 5e-2)  # trainer.hpp:13-20
    p = api.penalties()
    assert (p.rho_p, p.rho_q, p.rho_s, p.rho_f, p.rho_o) == (1e4, 1e4, 1e4, 1e3, 1e4)  # admm.hpp:12-18


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(api.BsgError):
        api.Block(0, 3)


def test_null_arguments_map_to_invalid_argument():
    lib = api.load_library()
    assert lib.bsg_create(0, 5, ctypes.byref(ctypes.c_void_p())) == api.BSG_ERR_INVALID_ARGUMENT
    assert b"feature" in lib.bsg_last_error()
