"""GPU parity of the rasterizer path (K1-K9) against the oracle, through the
C-ABI. Inputs are identical: the device stores FP32, so the oracle is fed the
same FP32-rounded parameters (HostCloud.narrowed()).

Bars (north star, BASELINE.json): integer paths bit-exact (visibility, rects,
FP64 depth, compositing order, tile keys); images max abs <= 1e-4; gradients
within a relative tolerance stated per test."""
import math

import numpy as np
import pytest

import _oracle as orc
from gpu_helpers import dev_cam, expected_pairs, gpu, new_block, rcfg, rel_err
from refcases import (HostCloud, aerial_scene, axis_camera, cloud_from_rows, empty_cloud, random_cloud, ref_camera,
                      splat_at)

pytestmark = gpu


def cases():
    """(name, cloud, camera) — reference test shapes plus a denser aerial block."""
    out = []
    for seed, size in ((77, 24), (78, 20), (81, 16), (90, 64), (91, 96)):
        out.append((f"random{seed}", random_cloud(40 if size < 64 else 400, seed).narrowed(), ref_camera(size)))
    cloud, cams = aerial_scene(20000, 160, 120, 4, 20.0, seed=5)
    for k, cam in enumerate(cams[:2]):
        out.append((f"aerial{k}", cloud.narrowed(), cam))
    return out


CASES = cases()


@pytest.mark.parametrize("name,cloud,cam", CASES, ids=[c[0] for c in CASES])
def test_projection_integer_paths_bit_exact(name, cloud, cam):
    b = new_block(cloud)
    got = b.project(dev_cam(cam))
    want = orc.project(cloud.oracle(), cam, orc.RenderConfig())
    assert np.array_equal(got["visible"], want["visible"])
    vis = want["visible"].astype(bool)
    assert np.array_equal(got["rect"][vis], want["rect"][vis])
    assert np.array_equal(got["depth"][vis].view(np.uint64), want["depth"][vis].view(np.uint64))
    assert np.array_equal(got["order"], want["order"])


@pytest.mark.parametrize("name,cloud,cam", CASES, ids=[c[0] for c in CASES])
def test_tile_keys_and_order_bit_exact(name, cloud, cam):
    want = orc.project(cloud.oracle(), cam, orc.RenderConfig())
    ek, er = expected_pairs(want, cam.width, cam.height)
    b = new_block(cloud)
    # global path (bsg_project): depth sort + tie fix-up + stable tile sort
    b.project(dev_cam(cam))
    tile, row = b.tile_pairs()
    assert np.array_equal(tile.astype(np.int64), ek)
    assert np.array_equal(row.astype(np.int64), er)
    # per-tile path (every render / training step): counts, atomic placement,
    # shared-memory (depth, row) sort per tile
    b.render(dev_cam(cam))
    tile, row = b.tile_pairs()
    assert np.array_equal(tile.astype(np.int64), ek)
    assert np.array_equal(row.astype(np.int64), er)


def test_per_tile_binning_falls_back_for_a_crowded_tile():
    """More pairs in one tile than the shared-memory sort takes (kTileSortCap
    = 2048): the first render switches to the global sort path after the tile
    scan, the next one takes it up front; order and image match both times."""
    g = np.random.default_rng(11)
    n = 6000
    cam = axis_camera(50, 8, 16)  # one 16x16 tile, principal point at its centre
    pos = np.column_stack([g.uniform(-0.4, 0.4, n), g.uniform(-0.4, 0.4, n), g.uniform(4.0, 6.0, n)])
    q = g.normal(size=(n, 4))
    cloud = HostCloud(np.arange(n, dtype=np.uint64), pos, q / np.linalg.norm(q, axis=1, keepdims=True),
                      np.full((n, 3), -4.0), g.uniform(0, 1, (n, 3)), g.normal(size=n) - 3.0)
    b = new_block(cloud)
    rgb, T, cnt = b.render(dev_cam(cam))
    want = orc.project(cloud.oracle(), cam, orc.RenderConfig())
    ek, er = expected_pairs(want, cam.width, cam.height)
    assert len(ek) > 4096  # well past the per-tile capacity
    tile, row = b.tile_pairs()
    assert np.array_equal(row.astype(np.int64), er)
    wrgb, wT, wn = orc.render(cloud.oracle(), cam, orc.RenderConfig())
    assert np.abs(rgb - wrgb).max() <= 1e-3
    rgb2, _, _ = b.render(dev_cam(cam))
    tile, row = b.tile_pairs()
    assert np.array_equal(row.astype(np.int64), er)
    assert np.abs(rgb2 - wrgb).max() <= 1e-3


@pytest.mark.parametrize("name,cloud,cam", CASES, ids=[c[0] for c in CASES])
def test_render_matches_oracle(name, cloud, cam):
    oc = orc.RenderConfig()
    oc.background = [0.2, 0.1, 0.05]
    b = new_block(cloud)
    rgb, T, n = b.render(dev_cam(cam), rcfg(oc))
    want, wT, wn = orc.render(cloud.oracle(), cam, oc)
    # FP32 blend: a contributor count may flip where T straddles the 1e-4
    # stop in FP32 vs FP64; such pixels differ by at most c*alpha*1e-4.
    flips = n != wn
    assert flips.mean() <= 1e-3
    assert np.abs(rgb - want)[~flips].max() <= 1e-4
    assert np.abs(T - wT)[~flips].max() <= 1e-5
    assert np.abs(rgb - want).max() <= 1e-3


def test_render_kats():
    """test_renderer.cpp:191-282 through the device path."""
    # empty cloud -> background, T = 1, n = 0
    b = new_block(empty_cloud())
    cam = axis_camera(50, 8, 16)
    oc = orc.RenderConfig()
    oc.background = [0.1, 0.2, 0.3]
    rgb, T, n = b.render(dev_cam(cam), rcfg(oc))
    assert np.allclose(rgb, [0.1, 0.2, 0.3], atol=1e-7) and np.all(T == 1.0) and np.all(n == 0)
    # single centred splat: C = 0.8 c, T = 0.2
    rows = []
    splat_at(rows, 1, [0, 0, 5], (0.9, 0.5, 0.25), 0.8)
    b = new_block(cloud_from_rows(rows))
    rgb, T, n = b.render(dev_cam(axis_camera(100, 8, 17)))
    assert np.allclose(rgb[8, 8], 0.8 * np.array([0.9, 0.5, 0.25]), atol=1e-6)
    assert abs(T[8, 8] - 0.2) < 1e-6 and n[8, 8] >= 1
    # alpha clamp
    rows = []
    splat_at(rows, 1, [0, 0, 5], (1.0, 1.0, 1.0), 0.9999)
    b = new_block(cloud_from_rows(rows))
    rgb, T, _ = b.render(dev_cam(axis_camera(100, 8, 17)))
    assert abs(rgb[8, 8, 0] - 0.99) < 1e-6 and abs(T[8, 8] - 0.01) < 1e-6
    # equal depth composites by index
    rows = []
    splat_at(rows, 1, [0, 0, 5], (0.8, 0, 0), 0.5)
    splat_at(rows, 2, [0, 0, 5], (0, 0, 0.8), 0.5)
    b = new_block(cloud_from_rows(rows))
    rgb, _, _ = b.render(dev_cam(axis_camera(100, 8, 17)))
    rgb2, _, _ = b.render(dev_cam(axis_camera(100, 8, 17)))
    assert np.array_equal(rgb, rgb2)
    assert abs(rgb[8, 8, 0] - 0.4) < 1e-6 and abs(rgb[8, 8, 2] - 0.2) < 1e-6
    # early stop after the third opaque splat
    rows = []
    for i in range(10):
        splat_at(rows, i + 1, [0, 0, 4 + 0.2 * i], (0.5, 0.5, 0.5), 0.9999)
    b = new_block(cloud_from_rows(rows))
    _, T, n = b.render(dev_cam(axis_camera(100, 8, 17)))
    assert n[8, 8] == 3 and T[8, 8] < 1e-4


def grad_close(got, want, rtol):
    """Norm-wise relative error per parameter group (FP32 atomics reorder sums)."""
    out = {}
    for k in ("g_pos", "g_rot", "g_ls", "g_feat", "g_op"):
        den = np.linalg.norm(want[k])
        out[k] = np.linalg.norm(got[k] - want[k]) / max(den, 1e-12)
    return out


BW_CASES = [c for c in CASES if not c[0].startswith("aerial1")]


@pytest.mark.parametrize("name,cloud,cam", BW_CASES, ids=[c[0] for c in BW_CASES])
def test_render_backward_matches_oracle(name, cloud, cam):
    rng = np.random.default_rng(3)
    gt = rng.uniform(0, 1, (cam.height, cam.width, 3))
    b = new_block(cloud)
    got = b.render_backward(dev_cam(cam), gt)
    want = orc.render_backward(cloud.oracle(), cam, gt, orc.RenderConfig())
    assert np.array_equal(got["visible"], want["visible"])
    # FP32 blend: per-pixel colour error ~1e-6 (MUFU exp, FP32 sums), so the
    # mean-absolute term is held to 1e-4 relative, the total loss to 2e-5.
    assert got["loss"] == pytest.approx(want["loss"], rel=2e-5)
    assert got["l1"] == pytest.approx(want["l1"], rel=1e-4)
    assert got["ssim"] == pytest.approx(want["ssim"], rel=1e-5, abs=1e-6)
    # Splats grazing the near plane (z ~ 0.01, only in the 30-degree aerial
    # cases; the reference has no frustum guard band) fold their image-space
    # gradient through 1/z^2 and 1/z^3 Jacobian terms that cancel to ~1e-5 of
    # their size. Their footprints are wide (>= kWideArea px), so the device
    # accumulates their image-space gradients in FP64 (deterministic; FP32
    # atomics gave 2-12% run-to-run); what remains is the FP32 per-pixel
    # arithmetic, ~4% on their position gradients. They are held to 6%; all
    # others to the 2e-3 norm-wise bar.
    proj = orc.project(cloud.oracle(), cam, orc.RenderConfig())
    grazing = proj["visible"].astype(bool) & (proj["depth"] < 1.0)
    errs = grad_close({k: (v[~grazing] if k.startswith("g_") else v) for k, v in got.items()},
                      {k: (v[~grazing] if k.startswith("g_") else v) for k, v in want.items()}, 1e-3)
    for k, e in errs.items():
        assert e <= 2e-3, (k, e)
    if grazing.any():
        errs = grad_close({k: (v[grazing] if k.startswith("g_") else v) for k, v in got.items()},
                          {k: (v[grazing] if k.startswith("g_") else v) for k, v in want.items()}, 1e-3)
        for k, e in errs.items():
            assert e <= 0.06, (k, e)
    # element-wise on the entries that carry the signal (non-grazing rows)
    for k in ("g_pos", "g_rot", "g_ls", "g_feat", "g_op"):
        gk, wk = got[k][~grazing], want[k][~grazing]
        big = np.abs(wk) > 1e-2 * np.abs(wk).max()
        if big.any():
            assert np.median(rel_err(gk[big], wk[big], 1e-12)) <= 1e-3
    sg = want["screen_grad_norm"][~grazing]
    assert np.linalg.norm(got["screen_grad_norm"][~grazing] - sg) <= 2e-3 * max(np.linalg.norm(sg), 1e-12)


def test_culled_rows_have_zero_gradients():
    """test_renderer.cpp:373-387."""
    rows = []
    splat_at(rows, 1, [0, 0, 5], (0.5, 0.5, 0.5), 0.7)
    splat_at(rows, 2, [0, 0, -5], (0.5, 0.5, 0.5), 0.7)
    c = cloud_from_rows(rows)
    b = new_block(c)
    got = b.render_backward(dev_cam(axis_camera(100, 8, 17)), np.full((17, 17, 3), 0.9))
    assert list(got["visible"]) == [1, 0]
    assert got["screen_grad_norm"][0] > 0 and got["screen_grad_norm"][1] == 0
    assert np.all(got["g_pos"][1] == 0) and got["g_op"][1] == 0 and got["g_op"][0] != 0


def test_zero_gradients_at_ground_truth():
    """test_renderer.cpp:316-332 (FP32: the device renders its own GT)."""
    c = random_cloud(8, 82).narrowed()
    cam = ref_camera(16)
    b = new_block(c)
    gt, _, _ = b.render(dev_cam(cam))
    got = b.render_backward(dev_cam(cam), gt)
    assert got["loss"] < 1e-6
    for k in ("g_pos", "g_rot", "g_ls", "g_feat", "g_op"):
        assert np.abs(got[k]).max() < 1e-4


def test_fd_gradients_through_device():
    """Acceptance criterion 1 (acceptance_main.cpp:67-129) through the device,
    at the reference's own bar: all 50 seeds (1000-1049), every parameter of
    every Gaussian, the device's FP32 analytic gradient against FP64 central
    differences of the oracle's loss, passing when err <= 1e-6 or rel <= 1e-3
    at h = 1e-5, re-probed at 1e-6 and 1e-7 (acceptance_main.cpp:101) --
    zero failures. The cloud is FP32-rounded so both sides see the same point.
    The camera position is Vec3(rng, rng, 5.5) drawn right to left (GCC's
    argument order, see refcases)."""
    from refcases import grad_check_cloud
    failed, checked = [], 0
    for s in range(50):
        rng = orc.Rng(1000 + s)
        c = grad_check_cloud(rng).narrowed()
        cy = rng.uniform_range(-0.5, 0.5)
        cx = rng.uniform_range(-0.5, 0.5)
        cam = orc.look_at([cx, cy, 5.5], [0, 0, 0], [0, 1, 0], 14, 14, 8, 8, 16, 16)
        gt = np.array([rng.uniform() for _ in range(16 * 16 * 3)]).reshape(16, 16, 3)
        got = new_block(c).render_backward(dev_cam(cam), gt)
        for name, gname in (("pos", "g_pos"), ("rot", "g_rot"), ("ls", "g_ls"), ("feat", "g_feat"), ("op", "g_op")):
            arr = getattr(c, name)
            for idx in np.ndindex(arr.shape):
                g = got[gname][idx]
                ok = False
                for h in (1e-5, 1e-6, 1e-7):
                    up, dn = c.copy(), c.copy()
                    getattr(up, name)[idx] += h
                    getattr(dn, name)[idx] -= h
                    fd = (orc.loss_value(orc.render(up.oracle(), cam, orc.RenderConfig())[0], gt, 0.2) -
                          orc.loss_value(orc.render(dn.oracle(), cam, orc.RenderConfig())[0], gt, 0.2)) / (2 * h)
                    err = abs(g - fd)
                    if err <= 1e-6 or err / max(abs(g), abs(fd), 1e-300) <= 1e-3:
                        ok = True
                        break
                checked += 1
                if not ok:
                    failed.append((s, name, idx, g, fd))
    assert checked == 50 * 8 * 14
    assert not failed, failed[:10]


def test_equal_depth_runs_keep_index_order():
    """Many splats with bit-identical FP64 depth (a fronto-parallel plane seen
    by an axis camera): the upper-32-bit depth sort + tie fix-up must give
    (depth, index) order; a run longer than 64 takes the full 64-bit path."""
    g = np.random.default_rng(7)
    for n_plane, n_other in ((40, 60), (300, 100)):
        rows = []
        for i in range(n_plane):
            splat_at(rows, i, [g.uniform(-0.5, 0.5), g.uniform(-0.5, 0.5), 5.0], (0.5, 0.2, 0.1), 0.5, -3.0)
        for i in range(n_other):
            splat_at(rows, n_plane + i, [g.uniform(-0.5, 0.5), g.uniform(-0.5, 0.5), g.uniform(4.0, 6.0)],
                     (0.1, 0.2, 0.5), 0.5, -3.0)
        c = cloud_from_rows(rows).narrowed()
        cam = axis_camera(100, 32, 64)
        b = new_block(c)
        got = b.project(dev_cam(cam))
        want = orc.project(c.oracle(), cam, orc.RenderConfig())
        assert np.array_equal(got["order"], want["order"])
        _per_tile_pairs_match(b, want, cam)


def _per_tile_pairs_match(b, want, cam):
    """The render's per-tile path (upper-32-bit bitonic sort + bounded tie
    fix-up + full-key re-sort of long runs) on the same cloud: tile keys and
    rows bit-exact against the reference bins re-expressed as tiles."""
    ek, er = expected_pairs(want, cam.width, cam.height)
    assert np.bincount(ek).max() <= 2048  # every tile fits the per-tile sort
    b.render(dev_cam(cam))
    assert b.last_binning() == "tile"
    tile, row = b.tile_pairs()
    assert np.array_equal(tile.astype(np.int64), ek)
    assert np.array_equal(row.astype(np.int64), er)


def plane_cluster_cloud(n, half_width, depth_spread, seed):
    """n splats on a plane facing the tilted reference camera, at depth 5 +-
    depth_spread (then rounded to f32 world positions), plus one far splat at
    depth ~5000 that stretches the depth span, so the 32-bit range-normalised
    depth key (~2^23 double ulps per bucket) merges many distinct FP64 depths."""
    cam = ref_camera(256)
    Rm = np.array(cam.R).reshape(3, 3)
    g = np.random.default_rng(seed)
    t = np.array(cam.t)
    pc = np.stack([g.uniform(-half_width, half_width, n), g.uniform(-half_width, half_width, n),
                   5.0 + g.uniform(-depth_spread, depth_spread, n)], 1)
    pc = np.vstack([pc, [[0.0, 0.0, 5000.0]]])
    pw = (pc - t) @ Rm
    rows = []
    for i, p in enumerate(pw):
        splat_at(rows, i, p, (0.5, 0.4, 0.3), 0.5, -4.0 if i < n else 1.0)
    return cloud_from_rows(rows).narrowed(), cam


@pytest.mark.parametrize("n,spread", [(20000, 2e-2), (6000, 1e-7)], ids=["short-runs", "long-runs"])
def test_depth_key_collisions_match_reference_order(n, spread):
    """Depth buckets holding several distinct FP64 depths: runs <= 64 go
    through the tie fix-up, longer out-of-order runs through the full 64-bit
    fall-back; both must reproduce renderer.cpp:86-89 bit-exactly."""
    cloud, cam = plane_cluster_cloud(n, 1.5, spread, 3)
    b = new_block(cloud)
    got = b.project(dev_cam(cam))
    want = orc.project(cloud.oracle(), cam, orc.RenderConfig())
    vis = want["visible"].astype(bool)
    assert vis.sum() > 0.9 * n
    assert np.array_equal(got["visible"], want["visible"])
    assert np.array_equal(got["order"], want["order"])
    _per_tile_pairs_match(b, want, cam)


def with_sh1(hc, seed, amp=0.5):
    """SH degree 1 copy (cloud.hpp:16-17): the band-0 colour plus random
    band-1 coefficients (channel-major, cloud.cpp:180-193)."""
    g = np.random.default_rng(seed)
    feat = np.concatenate([hc.feat[:, :3], amp * g.standard_normal((hc.n, 9))], 1)
    return HostCloud(hc.ids, hc.pos, hc.rot, hc.ls, feat, hc.op).narrowed()


def _bench_scene_sh1(n, w, h, seed):
    """The bench's aerial generator (5 degree tilt, no near-plane grazers: their
    FP32 conic cancellation is covered by the degree-0 30-degree cases) with
    band-1 features."""
    from paper_2405_13943_b200.scene import aerial_scene as bench_scene
    cl, cams = bench_scene(n, w, h, 4, 20.0, seed)
    hc = HostCloud(cl["ids"], cl["pos"], cl["rot"], cl["ls"], cl["feat"], cl["op"])
    c = cams[0]
    cam = orc.Camera()
    cam.fx, cam.fy, cam.cx, cam.cy = c.fx, c.fy, c.cx, c.cy
    cam.set_rotation_quat(list(c.q))
    cam.t = list(c.t)
    cam.width, cam.height = c.width, c.height
    return with_sh1(hc, 2), cam


SH1_CASES = [("random90-sh1", with_sh1(random_cloud(400, 90), 1), ref_camera(64)),
             ("aerial-sh1", *_bench_scene_sh1(20000, 160, 120, 5))]


@pytest.mark.parametrize("name,cloud,cam", SH1_CASES, ids=[c[0] for c in SH1_CASES])
def test_sh1_render_and_gradients(name, cloud, cam):
    """SH degree 1 through every device stage: view-dependent colour in the
    projection (bit-exact integer paths), the image, and the band-1 feature and
    view-direction position gradients of the fold."""
    assert cloud.fd == 12
    b = new_block(cloud)
    got = b.project(dev_cam(cam))
    want = orc.project(cloud.oracle(), cam, orc.RenderConfig())
    assert np.array_equal(got["visible"], want["visible"])
    assert np.array_equal(got["order"], want["order"])
    rgb, T, n = b.render(dev_cam(cam))
    wrgb, wT, wn = orc.render(cloud.oracle(), cam, orc.RenderConfig())
    flips = n != wn
    assert flips.mean() <= 1e-3
    assert np.abs(rgb - wrgb)[~flips].max() <= 1e-4
    gt = np.random.default_rng(4).uniform(0, 1, (cam.height, cam.width, 3))
    g = b.render_backward(dev_cam(cam), gt)
    w = orc.render_backward(cloud.oracle(), cam, gt, orc.RenderConfig())
    assert g["loss"] == pytest.approx(w["loss"], rel=2e-5)
    proj = want
    grazing = proj["visible"].astype(bool) & (proj["depth"] < 1.0)
    errs = grad_close({k: (v[~grazing] if k.startswith("g_") else v) for k, v in g.items()},
                      {k: (v[~grazing] if k.startswith("g_") else v) for k, v in w.items()}, 1e-3)
    for k, e in errs.items():
        assert e <= 2e-3, (k, e)
    assert g["g_feat"].shape[1] == 12 and np.abs(w["g_feat"][:, 3:]).max() > 0


@pytest.mark.parametrize("w,h,seed", [(16, 16, 1), (64, 48, 2), (256, 192, 3), (1024, 768, 4), (8, 12, 5)])
def test_image_loss_gradient_matches_ssim_with_gradient(w, h, seed):
    """dL/dC of the step (renderer.cpp:259-272) from the device's SSIM kernels
    against the FP64 oracle's ssim_with_gradient (ssim.cpp:138-185) on the
    same FP32-representable images: SSIM within 1e-6 absolute (the
    test_ssim.cpp gate), the loss within 1e-6 relative, and every dL/dC
    element within 1e-6 of the largest element (FP32 window sums; the L1 term
    is exact). Below 11x11 pixels SSIM = 1 with zero gradient (ssim.cpp:12-14)."""
    g = np.random.default_rng(seed)
    x = g.uniform(0, 1, (h, w, 3)).astype(np.float32).astype(np.float64)
    y = np.clip(x + 0.2 * g.standard_normal(x.shape), 0, 1).astype(np.float32).astype(np.float64)
    b = new_block(empty_cloud())
    l3, got = b.image_loss(x, y)
    s, ds = orc.ssim_with_gradient(x, y)
    want = np.sign(x - y) / (3.0 * w * h) - 0.2 * ds
    assert abs(l3[2] - s) <= 1e-6
    assert l3[0] == pytest.approx(orc.loss_value(x, y, 0.2), rel=1e-6)
    assert np.abs(got - want).max() <= 1e-6 * np.abs(want).max()
    if w < 11 or h < 11:
        assert s == 1.0 and not np.any(ds)
