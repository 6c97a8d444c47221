"""ctypes binding of the C-ABI in include/bsgpu.h (libbsgpu.so).

This is the Python mirror of the reference's operator surface for the hot
path: `Block` wraps one bsg context (one BlockTrainer's device state,
trainer.hpp:88-149) and exposes render / render_backward (renderer.hpp:71-81),
train_step (trainer.cpp:249-295) and the consensus round (admm.hpp:47-89).
There is no CPU fallback: if libbsgpu.so is missing or no sm_100 device is
present, construction raises.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BSG_LIB: developer override (A/B builds of the library); the default is the in-tree build.
LIB_PATH = os.environ.get("BSG_LIB") or os.path.join(_HERE, "lib", "libbsgpu.so")

BSG_OK = 0
BSG_ERR_INVALID_ARGUMENT = 1
BSG_ERR_CUDA = 2
BSG_ERR_NCCL = 3
BSG_ERR_STATE = 4
BSG_ERR_CAPACITY = 5
BSG_ERR_FORMAT = 6


class BsgError(RuntimeError):
    """std::runtime_error analogue (errors.hpp)."""


class InvalidArgument(ValueError):
    """blocksplat::InvalidArgument (errors.hpp:33-36)."""


class bsg_camera(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3), ("width", ctypes.c_uint32),
                ("height", ctypes.c_uint32)]


class bsg_render_config(ctypes.Structure):
    _fields_ = [("near_plane", ctypes.c_double), ("dilation", ctypes.c_double), ("alpha_clamp", ctypes.c_double),
                ("transmittance_stop", ctypes.c_double), ("sigma_extent", ctypes.c_double),
                ("background", ctypes.c_double * 3), ("lambda_", ctypes.c_double)]


class bsg_densify_config(ctypes.Structure):
    _fields_ = [("enabled", ctypes.c_int), ("interval", ctypes.c_uint32), ("stop_iteration", ctypes.c_uint64),
                ("grad_threshold", ctypes.c_double), ("prune_opacity", ctypes.c_double),
                ("split_scale_fraction", ctypes.c_double), ("split_shrink", ctypes.c_double),
                ("block_id", ctypes.c_uint32), ("global_initial_count", ctypes.c_uint64)]


class bsg_trainer_config(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_uint64), ("lr_position", ctypes.c_double),
                ("lr_position_decay", ctypes.c_double), ("lr_rotation", ctypes.c_double),
                ("lr_log_scale", ctypes.c_double), ("lr_features", ctypes.c_double), ("lr_opacity", ctypes.c_double),
                ("beta1", ctypes.c_double), ("beta2", ctypes.c_double), ("eps", ctypes.c_double),
                ("render", bsg_render_config), ("densify", bsg_densify_config)]


class bsg_penalties(ctypes.Structure):
    _fields_ = [("rho_p", ctypes.c_double), ("rho_q", ctypes.c_double), ("rho_s", ctypes.c_double),
                ("rho_f", ctypes.c_double), ("rho_o", ctypes.c_double)]


class bsg_round_args(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("relax", ctypes.c_int), ("n_reset", ctypes.c_size_t),
                ("reset_slots", ctypes.POINTER(ctypes.c_uint32)), ("diagnostics", ctypes.c_int)]


class bsg_round_result(ctypes.Structure):
    _fields_ = [("primal", ctypes.c_double), ("dual", ctypes.c_double), ("max_disagreement", ctypes.c_double),
                ("dual_mean_linf", ctypes.c_double), ("flipped", ctypes.c_uint64), ("ms", ctypes.c_double)]


class bsg_adapt_args(ctypes.Structure):
    _fields_ = [("mu", ctypes.c_double), ("tau_inc", ctypes.c_double), ("tau_dec", ctypes.c_double),
                ("freeze_iteration", ctypes.c_uint64), ("adaptive", ctypes.c_int), ("iteration", ctypes.c_uint64)]


class bsg_session_options(ctypes.Structure):
    _fields_ = [("total_iterations", ctypes.c_uint64), ("interval", ctypes.c_uint32), ("alpha", ctypes.c_double),
                ("mu", ctypes.c_double), ("tau_inc", ctypes.c_double), ("tau_dec", ctypes.c_double),
                ("freeze_iteration", ctypes.c_uint64), ("adaptive", ctypes.c_int), ("enabled", ctypes.c_int),
                ("rho", bsg_penalties), ("seed", ctypes.c_uint64), ("blocks", ctypes.c_uint32),
                ("expand_scale", ctypes.c_double), ("holdout", ctypes.c_uint32)]


class bsg_round_diag(ctypes.Structure):
    _fields_ = [("iteration", ctypes.c_uint64), ("primal", ctypes.c_double), ("dual", ctypes.c_double),
                ("rho", bsg_penalties), ("max_disagreement", ctypes.c_double), ("dual_mean_linf", ctypes.c_double),
                ("mean_loss", ctypes.c_double), ("shared_count", ctypes.c_uint64), ("global_count", ctypes.c_uint64),
                ("consensus_ms", ctypes.c_double)]


# (name, restype, argtypes) for every symbol declared in include/bsgpu.h.
_P = ctypes.c_void_p
_DP = ctypes.POINTER(ctypes.c_double)
_U32P = ctypes.POINTER(ctypes.c_uint32)
_U64P = ctypes.POINTER(ctypes.c_uint64)
_U8P = ctypes.POINTER(ctypes.c_uint8)
_FP = ctypes.POINTER(ctypes.c_float)
_SZ = ctypes.c_size_t
_SZP = ctypes.POINTER(ctypes.c_size_t)
SYMBOLS = [
    ("bsg_abi_version", ctypes.c_int, []),
    ("bsg_last_error", ctypes.c_char_p, []),
    ("bsg_default_render_config", None, [ctypes.POINTER(bsg_render_config)]),
    ("bsg_default_trainer_config", None, [ctypes.POINTER(bsg_trainer_config)]),
    ("bsg_default_penalties", None, [ctypes.POINTER(bsg_penalties)]),
    ("bsg_create", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]),
    ("bsg_destroy", ctypes.c_int, [_P]),
    ("bsg_upload_cloud", ctypes.c_int, [_P, _SZ, _U64P, _DP, _DP, _DP, _DP, _DP]),
    ("bsg_cloud_size", _SZ, [_P]),
    ("bsg_download_cloud", ctypes.c_int, [_P, _U64P, _DP, _DP, _DP, _DP, _DP]),
    ("bsg_encode_gspl", ctypes.c_int, [_P, _U8P, _SZ, _SZP]),
    ("bsg_save_model", ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _SZ, _U64P, _DP, _DP, _DP, _DP, _DP]),
    ("bsg_load_checkpoint", ctypes.c_int, [ctypes.c_char_p, _SZ, _U64P, _DP, _DP, _DP, _DP, _DP, _SZP,
                                            ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("bsg_decode_checkpoint", ctypes.c_int, [_U8P, _SZ, _SZ, _U64P, _DP, _DP, _DP, _DP, _DP, _SZP,
                                              ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("bsg_render", ctypes.c_int, [_P, ctypes.POINTER(bsg_camera), ctypes.POINTER(bsg_render_config), _DP, _DP, _U32P]),
    ("bsg_evaluate", ctypes.c_int, [_P, _SZ, ctypes.POINTER(bsg_camera), ctypes.POINTER(_DP), ctypes.c_uint32,
                                    ctypes.POINTER(bsg_render_config), _DP, _DP, _SZP, _DP, _DP]),
    ("bsg_render_backward", ctypes.c_int, [_P, ctypes.POINTER(bsg_camera), _DP, ctypes.POINTER(bsg_render_config), _DP,
                                            _DP, _DP, _DP, _DP, _DP, _DP, _U8P, _DP]),
    ("bsg_image_loss", ctypes.c_int, [_P, ctypes.c_uint32, ctypes.c_uint32, _DP, _DP, ctypes.POINTER(bsg_render_config),
                                       _DP, _DP]),
    ("bsg_project", ctypes.c_int, [_P, ctypes.POINTER(bsg_camera), ctypes.POINTER(bsg_render_config), _U8P, _DP,
                                    ctypes.POINTER(ctypes.c_int32), _U32P, _SZP]),
    ("bsg_tile_pairs", ctypes.c_int, [_P, _U32P, _U32P, _SZ, _SZP]),
    ("bsg_set_views", ctypes.c_int, [_P, _SZ, ctypes.POINTER(bsg_camera), ctypes.POINTER(_DP)]),
    ("bsg_trainer_init", ctypes.c_int, [_P, ctypes.POINTER(bsg_trainer_config)]),
    ("bsg_train_steps", ctypes.c_int, [_P, _SZ, _U32P, _DP]),
    ("bsg_train_step_host", ctypes.c_int, [_P, ctypes.POINTER(bsg_camera), _FP, _DP]),
    ("bsg_train_steps_host", ctypes.c_int, [_P, _SZ, ctypes.POINTER(bsg_camera), ctypes.POINTER(_FP), _DP]),
    ("bsg_train_steps_host_u8", ctypes.c_int, [_P, _SZ, ctypes.POINTER(bsg_camera), ctypes.POINTER(_U8P), _DP]),
    ("bsg_iteration", ctypes.c_uint64, [_P]),
    ("bsg_download_moments", ctypes.c_int, [_P, _DP, _DP]),
    ("bsg_upload_moments", ctypes.c_int, [_P, _DP, _DP, ctypes.c_uint64]),
    ("bsg_set_adam_sync_interval", ctypes.c_int, [_P, ctypes.c_uint32]),
    ("bsg_take_removed_ids", ctypes.c_int, [_P, _U64P, _SZ, _SZP]),
    ("bsg_take_new_ids", ctypes.c_int, [_P, _U64P, _SZ, _SZP]),
    ("bsg_shared_ids", ctypes.c_int, [_P, _U64P, _SZ, _SZP]),
    ("bsg_download_densify_stats", ctypes.c_int, [_P, _DP, _U32P]),
    ("bsg_set_shared", ctypes.c_int, [_P, _SZ, _U32P, _U32P, _U8P, _SZ, _U32P]),
    ("bsg_set_anchor", ctypes.c_int, [_P, _DP, _DP, ctypes.POINTER(bsg_penalties)]),
    ("bsg_set_penalties", ctypes.c_int, [_P, ctypes.POINTER(bsg_penalties)]),
    ("bsg_download_duals", ctypes.c_int, [_P, _DP]),
    ("bsg_download_anchor", ctypes.c_int, [_P, _DP]),
    ("bsg_upload_duals", ctypes.c_int, [_P, _DP]),
    ("bsg_download_consensus", ctypes.c_int, [_P, _DP]),
    ("bsg_apply_broadcast", ctypes.c_int, [_P, _DP, _SZ, _U32P, ctypes.c_double, ctypes.c_int]),
    ("bsg_nccl_unique_id", ctypes.c_int, [ctypes.POINTER(ctypes.c_uint8)]),
    ("bsg_comm_init", ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint8), ctypes.c_int, ctypes.c_int]),
    ("bsg_comm_init_local", ctypes.c_int, [ctypes.POINTER(_P), _SZ]),
    ("bsg_comm_init_host", ctypes.c_int, [_P, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
    ("bsg_set_round_timeout", ctypes.c_int, [_P, ctypes.c_double]),
    ("bsg_consensus_round", ctypes.c_int, [_P, ctypes.POINTER(bsg_round_args), ctypes.POINTER(bsg_round_result)]),
    ("bsg_consensus_round_async", ctypes.c_int, [_P, ctypes.POINTER(bsg_round_args), ctypes.POINTER(bsg_adapt_args)]),
    ("bsg_consensus_wait", ctypes.c_int, [_P, ctypes.POINTER(bsg_round_result), ctypes.POINTER(bsg_penalties)]),
    ("bsg_group_consensus_round", ctypes.c_int, [ctypes.POINTER(_P), _SZ, ctypes.POINTER(bsg_round_args),
                                                  ctypes.POINTER(bsg_round_result)]),
    ("bsg_plan_last_error", ctypes.c_char_p, []),
    ("bsg_plan_create", ctypes.c_int, [_SZ, _U64P, _DP, _SZ, _DP, ctypes.c_uint32, ctypes.c_double, ctypes.c_int,
                                        ctypes.c_int, ctypes.POINTER(_P)]),
    ("bsg_plan_destroy", None, [_P]),
    ("bsg_plan_block_sizes", ctypes.c_int, [_P, ctypes.c_uint32, _SZP, _SZP]),
    ("bsg_plan_block", ctypes.c_int, [_P, ctypes.c_uint32, _U64P, _U32P]),
    ("bsg_plan_boxes", ctypes.c_int, [_P, _DP, _DP, _DP, _DP]),
    ("bsg_plan_shared_count", _SZ, [_P]),
    ("bsg_plan_shared", ctypes.c_int, [_P, _U64P, _U32P, _U32P]),
    ("bsg_plan_block_shared", ctypes.c_int, [_P, ctypes.c_uint32, _SZP, _U32P, _U32P, _U8P]),
    ("bsg_driver_last_error", ctypes.c_char_p, []),
    ("bsg_view_sequence", ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint32, _SZ, _SZ, _U32P]),
    ("bsg_run_simulated", ctypes.c_int, [ctypes.c_int, _SZ, _U64P, _DP, _DP, _DP, _DP, _DP, _SZ,
                                          ctypes.POINTER(bsg_camera), ctypes.POINTER(_DP),
                                          ctypes.POINTER(bsg_trainer_config), ctypes.POINTER(bsg_session_options), _SZ,
                                          ctypes.POINTER(ctypes.c_int), _SZ, _U64P, _DP, _DP, _DP, _DP, _DP, _SZP,
                                          ctypes.POINTER(bsg_round_diag), _SZ, _SZP, _DP]),
    ("bsg_checked_build", ctypes.c_int, []),
    ("bsg_checked_probe", ctypes.c_int, [ctypes.c_int]),
    ("bsg_owners_create", ctypes.c_int, [ctypes.c_int, _SZ, _U64P, _U32P, ctypes.c_uint32, ctypes.POINTER(_P)]),
    ("bsg_owners_destroy", ctypes.c_int, [_P]),
    ("bsg_owners_size", _SZ, [_P]),
    ("bsg_owners_download", ctypes.c_int, [_P, _U64P, _U32P]),
    ("bsg_owners_remove", ctypes.c_int, [_P, ctypes.POINTER(_U64P), _SZP, _U32P, _U8P, _U32P, _SZ, _SZP, _U8P]),
    ("bsg_enable_stage_timing", ctypes.c_int, [_P, ctypes.c_int]),
    ("bsg_stage_count", ctypes.c_int, []),
    ("bsg_stage_name", ctypes.c_char_p, [ctypes.c_int]),
    ("bsg_stage_times", ctypes.c_int, [_P, _DP]),
    ("bsg_step_counters", ctypes.c_int, [_P, _U64P, _U64P, _U64P]),
    ("bsg_step_blend_evals", ctypes.c_uint64, [_P]),
    ("bsg_last_binning", ctypes.c_int, [_P]),
    ("bsg_launch_count", ctypes.c_uint64, [_P]),
    ("bsg_stream", _P, [_P]),
    ("bsg_synchronize", ctypes.c_int, [_P]),
]

_lib = None
HOST_ALLREDUCE = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                  ctypes.c_int)


def load_library(path=LIB_PATH):
    """Loads libbsgpu.so and binds every symbol; raises if anything is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise BsgError(f"{path} not built (run __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    for name, res, args in SYMBOLS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(status):
    if status == BSG_OK:
        return
    msg = _lib.bsg_last_error().decode()
    if status == BSG_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    raise BsgError(f"bsg status {status}: {msg}")


def _ptr(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype)) if a is not None else None


def make_camera(fx, fy, cx, cy, R, t, width, height):
    c = bsg_camera()
    c.fx, c.fy, c.cx, c.cy = float(fx), float(fy), float(cx), float(cy)
    R = np.asarray(R, dtype=np.float64).reshape(9)
    for k in range(9):
        c.R[k] = R[k]
    for k in range(3):
        c.t[k] = float(t[k])
    c.width, c.height = int(width), int(height)
    return c


def render_config(**kw):
    load_library()
    r = bsg_render_config()
    _lib.bsg_default_render_config(ctypes.byref(r))
    for k, v in kw.items():
        if k == "background":
            for i in range(3):
                r.background[i] = v[i]
        elif k == "lambda_" or k == "lam":
            r.lambda_ = v
        else:
            setattr(r, k, v)
    return r


def trainer_config(densify=None, **kw):
    """TrainerConfig defaults (trainer.hpp:13-62); densify: dict of
    DensifyConfig fields (e.g. {"enabled": 0})."""
    load_library()
    t = bsg_trainer_config()
    _lib.bsg_default_trainer_config(ctypes.byref(t))
    for k, v in kw.items():
        setattr(t, k, v)
    for k, v in (densify or {}).items():
        setattr(t.densify, k, v)
    return t


def penalties(**kw):
    load_library()
    p = bsg_penalties()
    _lib.bsg_default_penalties(ctypes.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


class Block:
    """One block's device state (BlockTrainer, trainer.hpp:88-149) on one GPU."""

    def __init__(self, device=0, feature_dim=3):
        load_library()
        self.fd = feature_dim
        self.D = 11 + feature_dim
        h = ctypes.c_void_p()
        _check(_lib.bsg_create(device, feature_dim, ctypes.byref(h)))
        self.h = h
        self._n = 0
        self.n_shared = 0
        self.n_slots = 0

    @property
    def n(self):
        """Rows in the device cloud (changes when densification runs)."""
        return int(_lib.bsg_cloud_size(self.h)) if self.h else self._n

    def close(self):
        if self.h:
            _lib.bsg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- parameters ----------------------------------------------------
    def upload_cloud(self, ids, pos, rot, ls, feat, op):
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        n = len(ids)
        pos, rot, ls = _f64(pos).reshape(n, 3), _f64(rot).reshape(n, 4), _f64(ls).reshape(n, 3)
        feat, op = _f64(feat).reshape(n, self.fd), _f64(op).reshape(n)
        _check(_lib.bsg_upload_cloud(self.h, n, _ptr(ids, ctypes.c_uint64), _ptr(pos, ctypes.c_double),
                                     _ptr(rot, ctypes.c_double), _ptr(ls, ctypes.c_double),
                                     _ptr(feat, ctypes.c_double), _ptr(op, ctypes.c_double)))
        self._n = n

    def download_cloud(self):
        n = self.n
        ids = np.zeros(n, np.uint64)
        pos, rot, ls = np.zeros((n, 3)), np.zeros((n, 4)), np.zeros((n, 3))
        feat, op = np.zeros((n, self.fd)), np.zeros(n)
        _check(_lib.bsg_download_cloud(self.h, _ptr(ids, ctypes.c_uint64), _ptr(pos, ctypes.c_double),
                                       _ptr(rot, ctypes.c_double), _ptr(ls, ctypes.c_double),
                                       _ptr(feat, ctypes.c_double), _ptr(op, ctypes.c_double)))
        return dict(ids=ids, pos=pos, rot=rot, ls=ls, feat=feat, op=op)

    def encode_gspl(self):
        """GSPL checkpoint payload of the device cloud (scene_io.cpp:48-59), encoded on the device."""
        ln = ctypes.c_size_t()
        _check(_lib.bsg_encode_gspl(self.h, None, 0, ctypes.byref(ln)))
        out = np.zeros(ln.value, np.uint8)
        _check(_lib.bsg_encode_gspl(self.h, _ptr(out, ctypes.c_uint8), ln.value, ctypes.byref(ln)))
        return out.tobytes()

    # ---- rendering -----------------------------------------------------
    def render(self, cam, cfg=None):
        H, W = cam.height, cam.width
        rgb, T, n = np.zeros((H, W, 3)), np.zeros((H, W)), np.zeros((H, W), np.uint32)
        _check(_lib.bsg_render(self.h, ctypes.byref(cam), ctypes.byref(cfg) if cfg else None,
                               _ptr(rgb, ctypes.c_double), _ptr(T, ctypes.c_double), _ptr(n, ctypes.c_uint32)))
        return rgb, T, n

    def evaluate(self, cams, gts, holdout_modulus=8, cfg=None):
        """evaluate (metrics.cpp:28-51) on the device: per-view PSNR / SSIM of
        the views with index % holdout_modulus == 0, and their means."""
        arr = (bsg_camera * len(cams))(*cams)
        keep = [_f64(g) for g in gts]
        ptrs = (_DP * len(cams))(*[_ptr(g, ctypes.c_double) for g in keep])
        p, q = np.zeros(max(len(cams), 1)), np.zeros(max(len(cams), 1))
        k, mp, ms = ctypes.c_size_t(), ctypes.c_double(), ctypes.c_double()
        _check(_lib.bsg_evaluate(self.h, len(cams), arr, ptrs, int(holdout_modulus), ctypes.byref(cfg) if cfg else None,
                                 _ptr(p, ctypes.c_double), _ptr(q, ctypes.c_double), ctypes.byref(k), ctypes.byref(mp),
                                 ctypes.byref(ms)))
        return dict(psnr=p[:k.value], ssim=q[:k.value], mean_psnr=mp.value, mean_ssim=ms.value)

    def render_backward(self, cam, gt, cfg=None):
        H, W = cam.height, cam.width
        gt = _f64(gt)
        if gt.shape != (H, W, 3):
            raise InvalidArgument("image dimension mismatch")
        n = self.n
        loss3 = np.zeros(3)
        g = dict(g_pos=np.zeros((n, 3)), g_rot=np.zeros((n, 4)), g_ls=np.zeros((n, 3)), g_feat=np.zeros((n, self.fd)),
                 g_op=np.zeros(n))
        sgn, vis, rend = np.zeros(n), np.zeros(n, np.uint8), np.zeros((H, W, 3))
        _check(_lib.bsg_render_backward(self.h, ctypes.byref(cam), _ptr(gt, ctypes.c_double),
                                        ctypes.byref(cfg) if cfg else None, _ptr(loss3, ctypes.c_double),
                                        *[_ptr(g[k], ctypes.c_double) for k in ("g_pos", "g_rot", "g_ls", "g_feat", "g_op")],
                                        _ptr(sgn, ctypes.c_double), _ptr(vis, ctypes.c_uint8),
                                        _ptr(rend, ctypes.c_double)))
        g.update(loss=loss3[0], l1=loss3[1], ssim=loss3[2], screen_grad_norm=sgn, visible=vis, rendered=rend)
        return g

    def image_loss(self, rendered, gt, cfg=None):
        """(loss, l1, ssim), dL/dC of the step's loss on given HxWx3 images."""
        rendered, gt = _f64(rendered), _f64(gt)
        H, W = rendered.shape[:2]
        if gt.shape != rendered.shape or rendered.shape != (H, W, 3):
            raise InvalidArgument("image dimension mismatch")
        l3, g = np.zeros(3), np.zeros((H, W, 3))
        _check(_lib.bsg_image_loss(self.h, W, H, _ptr(rendered, ctypes.c_double), _ptr(gt, ctypes.c_double),
                                   ctypes.byref(cfg) if cfg else None, _ptr(l3, ctypes.c_double),
                                   _ptr(g, ctypes.c_double)))
        return l3, g

    def project(self, cam, cfg=None):
        n = self.n
        vis, depth = np.zeros(n, np.uint8), np.zeros(n)
        rect = np.zeros((n, 4), np.int32)
        order = np.zeros(max(n, 1), np.uint32)
        V = ctypes.c_size_t()
        _check(_lib.bsg_project(self.h, ctypes.byref(cam), ctypes.byref(cfg) if cfg else None,
                                _ptr(vis, ctypes.c_uint8), _ptr(depth, ctypes.c_double),
                                _ptr(rect, ctypes.c_int32), _ptr(order, ctypes.c_uint32), ctypes.byref(V)))
        return dict(visible=vis, depth=depth, rect=rect, order=order[:V.value].astype(np.int64))

    def tile_pairs(self):
        P = ctypes.c_size_t()
        _check(_lib.bsg_tile_pairs(self.h, None, None, 0, ctypes.byref(P)))
        tile, row = np.zeros(max(P.value, 1), np.uint32), np.zeros(max(P.value, 1), np.uint32)
        _check(_lib.bsg_tile_pairs(self.h, _ptr(tile, ctypes.c_uint32), _ptr(row, ctypes.c_uint32), len(tile),
                                   ctypes.byref(P)))
        return tile[:P.value], row[:P.value]

    # ---- training ------------------------------------------------------
    def set_views(self, cams, gts):
        arr = (bsg_camera * len(cams))(*cams)
        self._gts = [_f64(g) for g in gts]
        ptrs = (_DP * len(cams))(*[_ptr(g, ctypes.c_double) for g in self._gts])
        _check(_lib.bsg_set_views(self.h, len(cams), arr, ptrs))
        self._gts = None

    def trainer_init(self, cfg=None):
        _check(_lib.bsg_trainer_init(self.h, ctypes.byref(cfg) if cfg else None))

    def train_steps(self, view_seq, want_losses=True):
        seq = np.ascontiguousarray(view_seq, dtype=np.uint32)
        losses = np.zeros(len(seq)) if want_losses else None
        _check(_lib.bsg_train_steps(self.h, len(seq), _ptr(seq, ctypes.c_uint32), _ptr(losses, ctypes.c_double)))
        return losses

    def train_step_host(self, cam, gt_f32):
        loss = ctypes.c_double()
        _check(_lib.bsg_train_step_host(self.h, ctypes.byref(cam), _ptr(gt_f32, ctypes.c_float), ctypes.byref(loss)))
        return loss.value

    def train_steps_host(self, cams, gts_f32):
        """n steps on host images (float32 HxWx3, pinned for overlap); returns the n losses."""
        n = len(cams)
        cam_arr = (bsg_camera * n)(*cams)
        keep = [np.ascontiguousarray(g, dtype=np.float32) for g in gts_f32]
        ptrs = (_FP * n)(*[_ptr(g, ctypes.c_float) for g in keep])
        out = np.zeros(n)
        _check(_lib.bsg_train_steps_host(self.h, n, cam_arr, ptrs, _ptr(out, ctypes.c_double)))
        return out

    def train_steps_host_u8(self, cams, gts_u8):
        """n steps on 8-bit host images (uint8 HxWx3, pinned for overlap); returns the n losses."""
        n = len(cams)
        cam_arr = (bsg_camera * n)(*cams)
        keep = [np.ascontiguousarray(g, dtype=np.uint8) for g in gts_u8]
        ptrs = (_U8P * n)(*[_ptr(g, ctypes.c_uint8) for g in keep])
        out = np.zeros(n)
        _check(_lib.bsg_train_steps_host_u8(self.h, n, cam_arr, ptrs, _ptr(out, ctypes.c_double)))
        return out

    def iteration(self):
        return _lib.bsg_iteration(self.h)

    def moments(self):
        m, v = np.zeros((self.D, self.n)), np.zeros((self.D, self.n))
        _check(_lib.bsg_download_moments(self.h, _ptr(m, ctypes.c_double), _ptr(v, ctypes.c_double)))
        return m, v

    def upload_moments(self, m, v, adam_step):
        """Optimizer state for a resume: m, v [D][n], the Adam step count."""
        m = np.ascontiguousarray(m, np.float64).reshape(self.D, self.n)
        v = np.ascontiguousarray(v, np.float64).reshape(self.D, self.n)
        _check(_lib.bsg_upload_moments(self.h, _ptr(m, ctypes.c_double), _ptr(v, ctypes.c_double), int(adam_step)))

    def set_adam_sync_interval(self, every):
        """Lazy Adam: every row caught up every `every` steps (1 = dense)."""
        _check(_lib.bsg_set_adam_sync_interval(self.h, int(every)))

    def _id_list(self, fn):
        n = ctypes.c_size_t()
        _check(fn(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros(max(n.value, 1), np.uint64)
        _check(fn(self.h, _ptr(out, ctypes.c_uint64), len(out), ctypes.byref(n)))
        return out[:n.value]

    def take_removed_ids(self):
        return self._id_list(_lib.bsg_take_removed_ids)

    def take_new_ids(self):
        return self._id_list(_lib.bsg_take_new_ids)

    def shared_ids(self):
        return self._id_list(_lib.bsg_shared_ids)

    def densify_stats(self):
        a, s = np.zeros(self.n), np.zeros(self.n, np.uint32)
        _check(_lib.bsg_download_densify_stats(self.h, _ptr(a, ctypes.c_double), _ptr(s, ctypes.c_uint32)))
        return a, s

    # ---- consensus -----------------------------------------------------
    def set_shared(self, rows, slots, first_owner, slot_owners):
        rows = np.ascontiguousarray(rows, np.uint32)
        slots = np.ascontiguousarray(slots, np.uint32)
        first = np.ascontiguousarray(first_owner, np.uint8)
        owners = np.ascontiguousarray(slot_owners, np.uint32)
        _check(_lib.bsg_set_shared(self.h, len(rows), _ptr(rows, ctypes.c_uint32), _ptr(slots, ctypes.c_uint32),
                                   _ptr(first, ctypes.c_uint8), len(owners), _ptr(owners, ctypes.c_uint32)))
        self.n_shared, self.n_slots = len(rows), len(owners)

    def set_anchor(self, z_rows, zprev_slots, rho):
        z = _f64(z_rows).reshape(self.n_shared, self.D)
        zp = _f64(zprev_slots).reshape(self.n_slots, self.D) if zprev_slots is not None else None
        _check(_lib.bsg_set_anchor(self.h, _ptr(z, ctypes.c_double), _ptr(zp, ctypes.c_double), ctypes.byref(rho)))

    def set_penalties(self, rho):
        _check(_lib.bsg_set_penalties(self.h, ctypes.byref(rho)))

    def duals(self):
        u = np.zeros((self.n_shared, self.D))
        _check(_lib.bsg_download_duals(self.h, _ptr(u, ctypes.c_double)))
        return u

    def anchor(self):
        z = np.zeros((self.n_shared, self.D))
        _check(_lib.bsg_download_anchor(self.h, _ptr(z, ctypes.c_double)))
        return z

    def consensus(self):
        z = np.zeros((self.n_slots, self.D))
        _check(_lib.bsg_download_consensus(self.h, _ptr(z, ctypes.c_double)))
        return z

    def apply_broadcast(self, z_slots, reset_slots, alpha, relax):
        z = _f64(z_slots).reshape(self.n_slots, self.D)
        rs = np.ascontiguousarray(reset_slots, np.uint32)
        _check(_lib.bsg_apply_broadcast(self.h, _ptr(z, ctypes.c_double), len(rs), _ptr(rs, ctypes.c_uint32) if len(rs) else None,
                                        float(alpha), 1 if relax else 0))

    def comm_init(self, uid, nranks, rank):
        buf = (ctypes.c_uint8 * 128)(*uid)
        _check(_lib.bsg_comm_init(self.h, buf, nranks, rank))

    def comm_init_host(self, allreduce, nranks, rank):
        """Host communicator (bsg_comm_init_host): allreduce(array, op) reduces
        the numpy view of the staging buffer in place (op "sum" / "max")."""
        def tramp(user, buf, count, dtype, op):
            try:
                ct = ctypes.c_double if dtype == 1 else ctypes.c_float
                arr = np.ctypeslib.as_array((ct * count).from_address(buf))
                allreduce(arr, "max" if op == 1 else "sum")
                return 0
            except Exception:
                return 1
        self._host_reduce = HOST_ALLREDUCE(tramp)  # kept alive with the block
        _check(_lib.bsg_comm_init_host(self.h, ctypes.cast(self._host_reduce, ctypes.c_void_p), None, nranks, rank))

    def set_round_timeout(self, seconds):
        _check(_lib.bsg_set_round_timeout(self.h, float(seconds)))

    def consensus_round(self, alpha, relax, reset_slots=(), diagnostics=False):
        a = _round_args(alpha, relax, reset_slots, diagnostics)
        r = bsg_round_result()
        _check(_lib.bsg_consensus_round(self.h, ctypes.byref(a), ctypes.byref(r)))
        return _round_dict(r)

    def consensus_round_async(self, alpha, relax, iteration=None, reset_slots=(), diagnostics=False, mu=10.0,
                              tau_inc=2.0, tau_dec=2.0, freeze_iteration=2000, adaptive=True):
        """Enqueue a round that overlaps the next train step (only its Adam
        waits). iteration=None: no penalty adaptation on the device."""
        self._round_args = _round_args(alpha, relax, reset_slots, diagnostics)  # keep alive until the call returns
        ad = None
        if iteration is not None:
            ad = bsg_adapt_args(mu, tau_inc, tau_dec, freeze_iteration, 1 if adaptive else 0, int(iteration))
        _check(_lib.bsg_consensus_round_async(self.h, ctypes.byref(self._round_args),
                                              ctypes.byref(ad) if ad is not None else None))

    def consensus_wait(self):
        r, rho = bsg_round_result(), bsg_penalties()
        _check(_lib.bsg_consensus_wait(self.h, ctypes.byref(r), ctypes.byref(rho)))
        d = _round_dict(r)
        d["rho"] = (rho.rho_p, rho.rho_q, rho.rho_s, rho.rho_f, rho.rho_o)
        return d

    # ---- measurement ---------------------------------------------------
    def enable_stage_timing(self, on=True):
        _check(_lib.bsg_enable_stage_timing(self.h, 1 if on else 0))

    def stage_times(self):
        k = _lib.bsg_stage_count()
        ms = np.zeros(k)
        _check(_lib.bsg_stage_times(self.h, _ptr(ms, ctypes.c_double)))
        return {_lib.bsg_stage_name(i).decode(): ms[i] for i in range(k)}

    def step_counters(self):
        v, p, l = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        _check(_lib.bsg_step_counters(self.h, ctypes.byref(v), ctypes.byref(p), ctypes.byref(l)))
        return dict(visible=v.value, pairs=p.value, launches=l.value, blend_evals=_lib.bsg_step_blend_evals(self.h))

    def last_binning(self):
        """'tile' (per-tile shared-memory sort) or 'global' for the last projection."""
        return {0: "tile", 1: "global"}[int(_lib.bsg_last_binning(self.h))]

    def launch_count(self):
        return _lib.bsg_launch_count(self.h)

    def stream(self):
        return _lib.bsg_stream(self.h)

    def synchronize(self):
        _check(_lib.bsg_synchronize(self.h))


def _round_args(alpha, relax, reset_slots, diagnostics):
    a = bsg_round_args()
    a.alpha = float(alpha)
    a.relax = 1 if relax else 0
    rs = np.ascontiguousarray(reset_slots, np.uint32)
    a.n_reset = len(rs)
    a._keep = rs
    a.reset_slots = _ptr(rs, ctypes.c_uint32) if len(rs) else None
    a.diagnostics = 1 if diagnostics else 0
    return a


def _round_dict(r):
    return dict(primal=r.primal, dual=r.dual, max_disagreement=r.max_disagreement,
                dual_mean_linf=r.dual_mean_linf, flipped=r.flipped, ms=r.ms)


def group_consensus_round(blocks, alpha, relax, reset_slots=(), diagnostics=False):
    """One consensus round over blocks held by this process (ascending block id)."""
    load_library()
    hs = (_P * len(blocks))(*[b.h.value for b in blocks])
    a = _round_args(alpha, relax, reset_slots, diagnostics)
    r = bsg_round_result()
    _check(_lib.bsg_group_consensus_round(hs, len(blocks), ctypes.byref(a), ctypes.byref(r)))
    return _round_dict(r)


class OwnerTable:
    """The master round's device owner table (bsg_owners_*):
    shared ids (ascending) with owner bitmasks over K <= 32 blocks."""

    def __init__(self, slot_ids, owner_masks, blocks, device=0):
        load_library()
        ids = np.ascontiguousarray(slot_ids, np.uint64)
        masks = np.ascontiguousarray(owner_masks, np.uint32)
        self.blocks = blocks
        h = ctypes.c_void_p()
        _check(_lib.bsg_owners_create(device, len(ids), _ptr(ids, ctypes.c_uint64), _ptr(masks, ctypes.c_uint32),
                                      blocks, ctypes.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            _lib.bsg_owners_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def table(self):
        n = _lib.bsg_owners_size(self.h)
        ids, masks = np.zeros(max(n, 1), np.uint64), np.zeros(max(n, 1), np.uint32)
        _check(_lib.bsg_owners_download(self.h, _ptr(ids, ctypes.c_uint64), _ptr(masks, ctypes.c_uint32)))
        return ids[:n], masks[:n]

    def remove(self, removed):
        """removed: per block, the ids it dropped this round. Returns (slots,
        classes, masks) of the touched slots and the per-id found flags."""
        lists = [np.ascontiguousarray(r, np.uint64) for r in removed]
        assert len(lists) == self.blocks
        ptrs = (_U64P * self.blocks)(*[_ptr(r, ctypes.c_uint64) for r in lists])
        ns = np.array([len(r) for r in lists], dtype=np.uintp)
        cap = int(_lib.bsg_owners_size(self.h)) + 1
        slot, cls, mask = np.zeros(cap, np.uint32), np.zeros(cap, np.uint8), np.zeros(cap, np.uint32)
        found = np.zeros(max(int(ns.sum()), 1), np.uint8)
        touched = ctypes.c_size_t()
        _check(_lib.bsg_owners_remove(self.h, ptrs, ns.ctypes.data_as(_SZP), _ptr(slot, ctypes.c_uint32),
                                      _ptr(cls, ctypes.c_uint8), _ptr(mask, ctypes.c_uint32), cap,
                                      ctypes.byref(touched), _ptr(found, ctypes.c_uint8)))
        k = touched.value
        return slot[:k], cls[:k], mask[:k], found[:int(ns.sum())]


def nccl_unique_id():
    load_library()
    buf = (ctypes.c_uint8 * 128)()
    _check(_lib.bsg_nccl_unique_id(buf))
    return bytes(buf)


class Plan:
    """Block partition + consensus slots (splitter.cpp:48-201, runtime.cpp:265-305),
    computed by the native host planner in libbsgpu.so."""

    def __init__(self, ids, pos, view_centers, k, scale, vertical_axis=1, midpoint_plane=False):
        load_library()
        ids = np.ascontiguousarray(ids, np.uint64)
        pos = _f64(pos).reshape(len(ids), 3)
        vc = _f64(view_centers).reshape(-1, 3) if len(view_centers) else np.zeros((0, 3))
        h = ctypes.c_void_p()
        st = _lib.bsg_plan_create(len(ids), _ptr(ids, ctypes.c_uint64), _ptr(pos, ctypes.c_double), len(vc),
                                  _ptr(vc, ctypes.c_double), k, float(scale), vertical_axis,
                                  1 if midpoint_plane else 0, ctypes.byref(h))
        if st != BSG_OK:
            msg = _lib.bsg_plan_last_error().decode()
            raise InvalidArgument(msg) if st == BSG_ERR_INVALID_ARGUMENT else BsgError(msg)
        self.h = h
        self.k = k

    def __del__(self):
        if getattr(self, "h", None):
            _lib.bsg_plan_destroy(self.h)
            self.h = None

    def block(self, b):
        ng, nv = ctypes.c_size_t(), ctypes.c_size_t()
        _lib.bsg_plan_block_sizes(self.h, b, ctypes.byref(ng), ctypes.byref(nv))
        ids, views = np.zeros(max(ng.value, 1), np.uint64), np.zeros(max(nv.value, 1), np.uint32)
        _lib.bsg_plan_block(self.h, b, _ptr(ids, ctypes.c_uint64), _ptr(views, ctypes.c_uint32))
        return ids[:ng.value], views[:nv.value]

    def boxes(self):
        k = self.k
        out = [np.zeros((k, 3)) for _ in range(4)]
        _lib.bsg_plan_boxes(self.h, *[_ptr(o, ctypes.c_double) for o in out])
        return dict(core_min=out[0], core_max=out[1], exp_min=out[2], exp_max=out[3])

    def shared(self):
        s = _lib.bsg_plan_shared_count(self.h)
        ids, cnt, first = np.zeros(max(s, 1), np.uint64), np.zeros(max(s, 1), np.uint32), np.zeros(max(s, 1), np.uint32)
        _lib.bsg_plan_shared(self.h, _ptr(ids, ctypes.c_uint64), _ptr(cnt, ctypes.c_uint32), _ptr(first, ctypes.c_uint32))
        return ids[:s], cnt[:s], first[:s]

    def block_shared(self, b):
        ids, _ = self.block(b)
        n = ctypes.c_size_t()
        rows, slots, first = (np.zeros(max(len(ids), 1), np.uint32), np.zeros(max(len(ids), 1), np.uint32),
                              np.zeros(max(len(ids), 1), np.uint8))
        _lib.bsg_plan_block_shared(self.h, b, ctypes.byref(n), _ptr(rows, ctypes.c_uint32), _ptr(slots, ctypes.c_uint32),
                                   _ptr(first, ctypes.c_uint8))
        return rows[:n.value], slots[:n.value], first[:n.value]


def view_sequence(seed, block_id, n_views, n_steps):
    """The C++ host BlockTrainer's view order (bsg_view_sequence)."""
    load_library()
    out = np.zeros(max(n_steps, 1), np.uint32)
    st = _lib.bsg_view_sequence(seed, block_id, n_views, n_steps, _ptr(out, ctypes.c_uint32))
    if st != BSG_OK:
        msg = _lib.bsg_driver_last_error().decode()
        raise InvalidArgument(msg) if st == BSG_ERR_INVALID_ARGUMENT else BsgError(msg)
    return out[:n_steps]


def session_options(total_iterations, interval=100, alpha=1.6, blocks=1, expand_scale=1.4, holdout=8, seed=0,
                    enabled=True, adaptive=True, rho=None):
    """SessionOptions + ConsensusConfig (runtime.hpp:109-115, admm.hpp:20-29) + plan arguments."""
    s = bsg_session_options()
    s.total_iterations, s.interval, s.alpha = total_iterations, interval, alpha
    s.mu, s.tau_inc, s.tau_dec, s.freeze_iteration = 10.0, 2.0, 2.0, 2000
    s.adaptive, s.enabled = int(adaptive), int(enabled)
    s.rho = rho if rho is not None else penalties()
    s.seed, s.blocks, s.expand_scale, s.holdout = seed, blocks, expand_scale, holdout
    return s


def run_simulated(cloud, cams, gts, trainer_cfg, session, devices=(0,)):
    """run_simulated (runtime.cpp:623-671) of the native host layer: plan_cluster
    + K device BlockTrainers + device consensus rounds. Returns (model, rounds, wall_s)."""
    load_library()
    ids = np.ascontiguousarray(cloud["ids"], np.uint64)
    n = len(ids)
    fd = np.asarray(cloud["feat"]).reshape(n, -1).shape[1]
    arrs = [_f64(cloud[k]) for k in ("pos", "rot", "ls", "feat", "op")]
    cam_arr = (bsg_camera * len(cams))(*cams)
    gts = [_f64(g) for g in gts]
    gptr = (_DP * len(gts))(*[_ptr(g, ctypes.c_double) for g in gts])
    cap = 16 * n + 1024  # densification grows the model
    out_ids = np.zeros(cap, np.uint64)
    outs = [np.zeros((cap, 3)), np.zeros((cap, 4)), np.zeros((cap, 3)), np.zeros((cap, fd)), np.zeros(cap)]
    n_out = ctypes.c_size_t()
    max_rounds = int(session.total_iterations // max(session.interval, 1)) + 2
    rounds = (bsg_round_diag * max_rounds)()
    nr, wall = ctypes.c_size_t(), ctypes.c_double()
    dev = (ctypes.c_int * len(devices))(*devices)
    st = _lib.bsg_run_simulated(fd, n, _ptr(ids, ctypes.c_uint64), *[_ptr(a, ctypes.c_double) for a in arrs],
                                len(cams), cam_arr, gptr, ctypes.byref(trainer_cfg), ctypes.byref(session),
                                len(devices), dev, cap, _ptr(out_ids, ctypes.c_uint64),
                                *[_ptr(o, ctypes.c_double) for o in outs], ctypes.byref(n_out), rounds, max_rounds,
                                ctypes.byref(nr), ctypes.byref(wall))
    if st != BSG_OK:
        msg = _lib.bsg_driver_last_error().decode()
        raise InvalidArgument(msg) if st == BSG_ERR_INVALID_ARGUMENT else BsgError(msg)
    m = n_out.value
    model = dict(ids=out_ids[:m], pos=outs[0][:m], rot=outs[1][:m], ls=outs[2][:m], feat=outs[3][:m], op=outs[4][:m])
    rl = []
    for j in range(min(nr.value, max_rounds)):
        r = rounds[j]
        rl.append(dict(iteration=r.iteration, primal=r.primal, dual=r.dual,
                       rho=(r.rho.rho_p, r.rho.rho_q, r.rho.rho_s, r.rho.rho_f, r.rho.rho_o),
                       max_disagreement=r.max_disagreement, dual_mean_linf=r.dual_mean_linf, mean_loss=r.mean_loss,
                       shared_count=r.shared_count, global_count=r.global_count, consensus_ms=r.consensus_ms))
    return model, rl, wall.value


class FormatError(RuntimeError):
    """blocksplat::FormatError (errors.hpp:10-31); .code is the FormatErrorCode name."""

    CODES = ("BadMagic", "UnsupportedVersion", "TruncatedSection", "UnknownSection", "TruncatedBuffer",
             "CountOverflow", "NonMonotoneIds", "BadHeader")

    def __init__(self, code, msg):
        super().__init__(f"{self.CODES[code]}: {msg}")
        self.code = self.CODES[code]


def _driver_check(status, fcode=None):
    if status == BSG_OK:
        return
    msg = _lib.bsg_driver_last_error().decode()
    if status == BSG_ERR_FORMAT:
        raise FormatError(fcode.value, msg)
    if status == BSG_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    raise BsgError(f"bsg status {status}: {msg}")


def save_model(path, cloud):
    """model.dogs (main.cpp:353-357): DOGS container with the f32-narrowed model as its GSPL section."""
    load_library()
    ids = np.ascontiguousarray(cloud["ids"], np.uint64)
    n = len(ids)
    fd = np.asarray(cloud["feat"]).reshape(n, -1).shape[1] if n else int(cloud.get("fd", 3))
    arrs = [_f64(cloud[k]) for k in ("pos", "rot", "ls", "feat", "op")]
    _driver_check(_lib.bsg_save_model(os.fsencode(path), fd, n, _ptr(ids, ctypes.c_uint64),
                                      *[_ptr(a, ctypes.c_double) for a in arrs]))


def _checkpoint(call):
    n, fd, fc = ctypes.c_size_t(), ctypes.c_int(), ctypes.c_int(-1)
    _driver_check(call(0, None, None, None, None, None, None, ctypes.byref(n), ctypes.byref(fd), ctypes.byref(fc)), fc)
    m, f = n.value, fd.value
    ids = np.zeros(max(m, 1), np.uint64)
    outs = [np.zeros((max(m, 1), w)) for w in (3, 4, 3, f)] + [np.zeros(max(m, 1))]
    _driver_check(call(m, _ptr(ids, ctypes.c_uint64), *[_ptr(o, ctypes.c_double) for o in outs], ctypes.byref(n),
                       ctypes.byref(fd), ctypes.byref(fc)), fc)
    return dict(ids=ids[:m], pos=outs[0][:m], rot=outs[1][:m], ls=outs[2][:m], feat=outs[3][:m], op=outs[4][:m])


def load_checkpoint(path):
    """GSPL checkpoint of a DOGS container file (runtime.cpp:273-275), as FP64 arrays."""
    load_library()
    p = os.fsencode(path)
    return _checkpoint(lambda cap, *a: _lib.bsg_load_checkpoint(p, cap, *a))


def decode_checkpoint(data):
    """GSPL checkpoint of DOGS container bytes (decode_scene, scene_io.cpp:134-176)."""
    load_library()
    buf = np.frombuffer(bytes(data), np.uint8).copy()
    ptr = _ptr(buf, ctypes.c_uint8) if len(buf) else None
    return _checkpoint(lambda cap, *a: _lib.bsg_decode_checkpoint(ptr, len(buf), cap, *a))
