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


gpu = pytest.mark.gpu
