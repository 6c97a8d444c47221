"""Glue between oracle fixtures and the device C-ABI (tests only)."""
import numpy as np
import pytest

from paper_2405_13943_b200 import api


def dev_cam(cam):
    """oracle Camera -> bsg_camera with the identical FP64 R, t."""
    return api.make_camera(cam.fx, cam.fy, cam.cx, cam.cy, cam.R, cam.t, cam.width, cam.height)


def upload(block, hc):
    block.upload_cloud(hc.ids, hc.pos, hc.rot, hc.ls, hc.feat, hc.op)


def new_block(hc, device=0):
    b = api.Block(device, hc.fd)
    upload(b, hc)
    return b


def rcfg(oc):
    """oracle RenderConfig -> bsg_render_config."""
    return api.render_config(near_plane=oc.near_plane, dilation=oc.dilation, alpha_clamp=oc.alpha_clamp,
                             transmittance_stop=oc.transmittance_stop, sigma_extent=oc.sigma_extent,
                             background=list(oc.background), lambda_=oc.lambda_)


def expected_pairs(proj, W, H, tile=16):
    """Tile keys the reference implies: every splat in (depth, index) order
    duplicated into each 16x16 tile its rect overlaps, stably sorted by tile."""
    tiles_x = (W + tile - 1) // tile
    keys, rows = [], []
    for r in proj["order"]:
        x0, x1, y0, y1 = proj["rect"][r]
        for ty in range(y0 // tile, y1 // tile + 1):
            for tx in range(x0 // tile, x1 // tile + 1):
                keys.append(ty * tiles_x + tx)
                rows.append(r)
    keys = np.array(keys, dtype=np.int64)
    rows = np.array(rows, dtype=np.int64)
    o = np.argsort(keys, kind="stable")
    return keys[o], rows[o]


def rel_err(a, b, floor):
    return np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)


def check_adam_trajectory(got, want, grads, cfg, steps, min_conf=0.05):
    """Device parameters after `steps` Adam steps vs the oracle trainer's, with
    a bound derived from the update rule (trainer.cpp:120-131) rather than a
    blanket tolerance. A step moves a coordinate by lr * m_hat / (sqrt(v_hat) +
    eps): by lr * sign(g) on the first step, and later by an amount that
    depends on the ratios of the steps' gradients, so an FP32 gradient error e
    moves it by ~e * lr. Hence
    - every coordinate within 2 * lr * steps (the sign-flip bound of tiny gradients);
    - "confident" coordinates, whose oracle gradient is >= 1% of the group's
      largest at every step, within 2e-2 * lr * steps (at least min_conf of the
      coordinates that saw a gradient must be confident);
    - coordinates with an exactly zero gradient at every step unchanged.
    got/want: dicts pos/rot/ls/feat/op; grads: per step, the oracle's
    render_backward outputs before that step (penalty-free blocks)."""
    n = len(np.asarray(want["pos"]).reshape(-1, 3))
    groups = (("pos", "g_pos", cfg.lr_position), ("rot", "g_rot", cfg.lr_rotation), ("ls", "g_ls", cfg.lr_log_scale),
              ("feat", "g_feat", cfg.lr_features), ("op", "g_op", cfg.lr_opacity))
    for name, gname, lr in groups:
        g, w = np.asarray(got[name]).reshape(n, -1), np.asarray(want[name]).reshape(n, -1)
        err = np.abs(g - w)
        slack = 2e-6 * (1.0 + np.abs(w))  # FP32 storage of x
        assert np.all(err <= 2 * lr * steps + slack), (name, err.max())
        conf = np.ones(g.shape, bool)
        touched = np.zeros(g.shape, bool)
        for gr in grads:
            a = np.abs(np.asarray(gr[gname]).reshape(g.shape))
            conf &= a >= 1e-2 * a.max()
            touched |= a > 0
        assert conf.sum() >= min_conf * touched.sum(), (name, conf.sum(), touched.sum())
        assert np.all(err[conf] <= 2e-2 * lr * steps + slack[conf]), (name, err[conf].max())
        assert np.all(err[~touched] <= slack[~touched]), name


gpu = pytest.mark.gpu
