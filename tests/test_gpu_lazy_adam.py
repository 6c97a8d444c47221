"""Lazy Adam is the dense Adam, bit for bit (trainer.cpp:120-131 applies the
update to every row every step; the device skips rows without a gradient or
penalty and replays the skipped zero-gradient steps when the row is next
needed).

Two clusters of Gaussians, far apart, one camera on each. Both blocks start
from the same parameters and optimizer state (bsg_upload_moments, t = 5) and
train 40 steps on camera B only, so cluster A never receives a gradient:
- block D syncs every step (`bsg_set_adam_sync_interval(1)`: every row's
  zero-gradient step applied in the Adam kernels' file, the dense update);
- block L uses interval 32 (default 16): cluster A is replayed 27 steps at
  once at t = 32 (materialize), then 13 steps inside the projection kernel
  (a file compiled with --fmad=false) when camera A is rendered at t = 45,
  and the rows outside camera A's view by the read's materialize.
Cluster A's parameters, moments and camera A's image must then be
bit-identical between the blocks. (Cluster B's rows are not compared: the
blend backward accumulates gradients with FP32 atomics, whose order is not
deterministic across runs.)"""
import numpy as np
import pytest

import _oracle as orc
from gpu_helpers import dev_cam, gpu
from paper_2405_13943_b200 import api

pytestmark = gpu

SIZE = 64


def two_clusters(fd, n_each=1500, seed=11):
    g = np.random.default_rng(seed)
    n = 2 * n_each
    centre = np.repeat(np.array([[-20.0, 0.0, 0.0], [20.0, 0.0, 0.0]]), n_each, 0)
    pos = centre + g.uniform(-1.5, 1.5, (n, 3))
    q = g.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[q[:, 0] < 0] *= -1
    ls = g.uniform(-2.5, -0.8, (n, 3))
    ls[::3] = ls[::3] * np.array([1.0, 0.6, 1.3])  # anisotropic rows: rotation gradients are real
    feat = g.uniform(0.0, 3.0, (n, fd))
    op = g.uniform(-1.5, 2.0, n)
    return dict(ids=np.arange(n, dtype=np.uint64), pos=pos, rot=q, ls=ls, feat=feat, op=op), n_each


def cams():
    a = orc.look_at([-20.0, 0.3, -6.0], [-20.0, 0.0, 0.0], [0.0, 1.0, 0.0], 1.1 * SIZE, 1.1 * SIZE, SIZE / 2.0,
                    SIZE / 2.0, SIZE, SIZE)
    b = orc.look_at([20.0, 0.3, -6.0], [20.0, 0.0, 0.0], [0.0, 1.0, 0.0], 1.1 * SIZE, 1.1 * SIZE, SIZE / 2.0,
                    SIZE / 2.0, SIZE, SIZE)
    return dev_cam(a), dev_cam(b)


def run(cloud, fd, m0, v0, sync, steps=40):
    ca, cb = cams()
    b = api.Block(0, fd)
    try:
        b.upload_cloud(cloud["ids"], cloud["pos"], cloud["rot"], cloud["ls"], cloud["feat"], cloud["op"])
        gt = np.full((SIZE, SIZE, 3), 0.25)
        b.set_views([ca, cb], [gt, gt])
        b.trainer_init(api.trainer_config(iterations=200, densify={"enabled": 0}))
        b.upload_moments(m0, v0, 5)
        b.set_adam_sync_interval(sync)
        b.train_steps([1] * steps, want_losses=False)
        img = b.render(ca)
        m, v = b.moments()
        x = b.download_cloud()
        return img, m, v, x
    finally:
        b.close()


@pytest.mark.parametrize("fd", [3, 12])
def test_lazy_adam_is_dense_adam_bitwise(fd):
    cloud, na = two_clusters(fd)
    D = 11 + fd
    n = 2 * na
    g = np.random.default_rng(5)
    # moments as after a few steps: |m_hat / sqrt(v_hat)| ~ 1, so every replayed step moves x
    m0 = (g.normal(size=(D, n)) * 1e-3).astype(np.float32).astype(np.float64)
    v0 = (g.uniform(0.5, 2.0, (D, n)) * 1e-6).astype(np.float32).astype(np.float64)
    img_l, m_l, v_l, x_l = run(cloud, fd, m0, v0, 32)
    img_d, m_d, v_d, x_d = run(cloud, fd, m0, v0, 1)
    a = slice(0, na)
    for name in ("pos", "rot", "ls", "feat", "op"):
        xl, xd = np.asarray(x_l[name])[a], np.asarray(x_d[name])[a]
        assert np.array_equal(xl, xd), (name, np.abs(xl - xd).max(), int((xl != xd).sum()))
    assert np.array_equal(m_l[:, a], m_d[:, a]) and np.array_equal(v_l[:, a], v_d[:, a])
    # the replay really moved cluster A (not a vacuous comparison) ...
    assert np.abs(np.asarray(x_l["pos"])[a] - cloud["pos"][a]).max() > 2e-4
    assert np.all(np.abs(m_l[:, a]) < np.abs(m0[:, a]) + 1e-30)  # zero-gradient steps only shrink m
    # ... camera A sees it, and both blocks render the same image
    assert img_l[0].std() > 1e-3
    for k in range(3):  # rgb, T, n
        assert np.array_equal(img_l[k], img_d[k]), k
    # cluster B trained in both (its values differ only by the atomics' order)
    assert np.abs(np.asarray(x_l["pos"])[na:] - cloud["pos"][na:]).max() > 1e-3
