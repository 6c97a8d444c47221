"""Pins the oracle (CPU FP64 restatement) to the reference's own known-answer
tests. Each test cites the reference test it restates; tolerances are the
reference's. CPU only."""
import math

import numpy as np
import pytest

import _oracle as orc
from refcases import (SH0, HostCloud, axis_camera, cloud_from_rows, empty_cloud, grad_check_cloud, logit,
                      random_bundle, random_cloud, random_image, scalar_cloud, splat_at, ref_camera, dapprox)


def cfg(**kw):
    c = orc.RenderConfig()
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def one_gaussian(pos, cov_scale=1.0):
    # Sigma = cov_scale * I  <=>  identity rotation, log_scale = log(sqrt(cov_scale)).
    ls = 0.5 * math.log(cov_scale)
    return cloud_from_rows([(0, list(pos), [1.0, 0, 0, 0], [ls] * 3, [0, 0, 0], 0.0)])


# ------------------------------------------------------------ test_renderer.cpp
def test_on_axis_projection():  # test_renderer.cpp:139-149
    p = orc.project(one_gaussian([0, 0, 5]).oracle(), axis_camera(100, 32, 64), cfg())
    assert p["visible"][0]
    assert tuple(p["mean2d"][0]) == (32.0, 32.0)
    assert p["depth"][0] == 5.0
    assert p["cov2d"][0, 0, 0] == pytest.approx(400.3, rel=1e-12)
    assert p["cov2d"][0, 1, 1] == pytest.approx(400.3, rel=1e-12)
    assert p["cov2d"][0, 0, 1] == 0.0


def test_near_plane_cull():  # test_renderer.cpp:151-156
    cam = axis_camera(100, 32, 64)
    assert not orc.project(one_gaussian([0, 0, -1]).oracle(), cam, cfg())["visible"][0]
    assert not orc.project(one_gaussian([0, 0, 0.005]).oracle(), cam, cfg())["visible"][0]
    assert orc.project(one_gaussian([0, 0, 0.02], 1e-6).oracle(), cam, cfg())["visible"][0]


def test_off_image_cull():  # test_renderer.cpp:158-162
    assert not orc.project(one_gaussian([40, 0, 5], 0.01).oracle(), axis_camera(100, 32, 64), cfg())["visible"][0]


def test_cov2d_matches_fd_jacobian():  # test_renderer.cpp:164-189
    cam = ref_camera(48)
    R = cam.R
    t = np.array(cam.t)
    rng = orc.Rng(31)
    checked = 0
    for trial in range(12):
        z = rng.uniform_range(-1, 1); y = rng.uniform_range(-1, 1); x = rng.uniform_range(-1, 1)
        q = rng.random_unit_quat()
        l3 = rng.uniform_range(-2, -0.5); l2 = rng.uniform_range(-2, -0.5); l1 = rng.uniform_range(-2, -0.5)
        c = cloud_from_rows([(0, [x, y, z], q, [l1, l2, l3], [0, 0, 0], 0.0)])
        p = orc.project(c.oracle(), cam, cfg())
        if not p["visible"][0]:
            continue
        Rq = orc.quat_to_rotation(q)
        S = np.diag(np.exp([l1, l2, l3]))
        sigma = (Rq @ S) @ (Rq @ S).T
        pc = R @ np.array([x, y, z]) + t
        h = 1e-6
        proj = lambda v: np.array([cam.fx * v[0] / v[2] + cam.cx, cam.fy * v[1] / v[2] + cam.cy])
        J = np.stack([(proj(pc + h * e) - proj(pc - h * e)) / (2 * h) for e in np.eye(3)], 1)
        A = J @ R
        ref = A @ sigma @ A.T + 0.3 * np.eye(2)
        assert np.abs(p["cov2d"][0] - ref).max() < 1e-5 * np.linalg.norm(ref)
        checked += 1
    assert checked > 0


def test_empty_cloud_renders_background():  # test_renderer.cpp:191-202
    color, T, n = orc.render(empty_cloud().oracle(), axis_camera(50, 8, 16), cfg(background=[0.1, 0.2, 0.3]))
    assert np.all(color == np.array([0.1, 0.2, 0.3]))
    assert np.all(T == 1.0) and np.all(n == 0)


def test_single_centered_splat():  # test_renderer.cpp:204-216
    rows = []
    rgb = (0.9, 0.5, 0.25)
    splat_at(rows, 1, [0, 0, 5], rgb, 0.8)
    color, T, n = orc.render(cloud_from_rows(rows).oracle(), axis_camera(100, 8, 17), cfg())
    assert color[8, 8] == pytest.approx(0.8 * np.array(rgb), rel=1e-12)
    assert T[8, 8] == pytest.approx(0.2, rel=1e-12)
    assert n[8, 8] >= 1


def test_alpha_clamp():  # test_renderer.cpp:218-227
    rows = []
    splat_at(rows, 1, [0, 0, 5], [1.0, 1.0, 1.0], 0.9999)
    color, T, _ = orc.render(cloud_from_rows(rows).oracle(), axis_camera(100, 8, 17), cfg())
    assert color[8, 8, 0] == pytest.approx(0.99, rel=1e-10)
    assert T[8, 8] == pytest.approx(0.01, rel=1e-8)


def brute_force(cloud, cam, c):
    """Independent compositor (test_renderer.cpp:68-135): every splat, rect test per pixel."""
    p = orc.project(cloud.oracle(), cam, c)
    order = p["order"]
    H, W = cam.height, cam.width
    out = np.zeros((H, W, 3))
    T = np.ones((H, W))
    wsum = np.zeros((H, W))
    for y in range(H):
        for x in range(W):
            t = 1.0
            col = np.zeros(3)
            ws = 0.0
            for i in order:
                x0, x1, y0, y1 = p["rect"][i]
                if x < x0 or x > x1 or y < y0 or y > y1:
                    continue
                if t < c.transmittance_stop:
                    break
                d = np.array([x, y]) - p["mean2d"][i]
                q = d @ np.linalg.inv(p["cov2d"][i]) @ d
                a = min(p["opacity"][i] * math.exp(-0.5 * q), c.alpha_clamp)
                col += p["color"][i] * (a * t)
                ws += a * t
                t *= 1 - a
            out[y, x] = col + t * np.array(c.background)
            T[y, x] = t
            wsum[y, x] = ws
    return out, T, wsum


def test_render_matches_brute_force():  # test_renderer.cpp:229-242
    c = random_cloud(24, 77)
    cam = ref_camera(24)
    rc = cfg(background=[0.2, 0.1, 0.05])
    color, T, _ = orc.render(c.oracle(), cam, rc)
    want, wT, _ = brute_force(c, cam, rc)
    assert np.abs(color - want).max() < 1e-10
    np.testing.assert_allclose(T, wT, rtol=1e-10)


def test_weights_plus_transmittance_is_one():  # test_renderer.cpp:244-255
    c = random_cloud(30, 78)
    cam = ref_camera(20)
    _, T, _ = orc.render(c.oracle(), cam, cfg())
    _, wT, ws = brute_force(c, cam, cfg())
    assert np.abs(ws + wT - 1.0).max() < 1e-12
    assert T.min() >= 0.0 and T.max() <= 1.0


def test_equal_depth_composites_by_index():  # test_renderer.cpp:257-270
    rows = []
    splat_at(rows, 1, [0, 0, 5], [0.8, 0, 0], 0.5)
    splat_at(rows, 2, [0, 0, 5], [0, 0, 0.8], 0.5)
    c = cloud_from_rows(rows).oracle()
    a = orc.render(c, axis_camera(100, 8, 17), cfg())[0]
    b = orc.render(c, axis_camera(100, 8, 17), cfg())[0]
    assert np.array_equal(a, b)
    assert a[8, 8, 0] == pytest.approx(0.4, rel=1e-12)
    assert a[8, 8, 2] == pytest.approx(0.2, rel=1e-12)


def test_early_stop():  # test_renderer.cpp:272-282
    rows = []
    for i in range(10):
        splat_at(rows, i + 1, [0, 0, 4 + 0.2 * i], [0.5] * 3, 0.9999)
    _, T, n = orc.render(cloud_from_rows(rows).oracle(), axis_camera(100, 8, 17), cfg())
    assert n[8, 8] == 3
    assert T[8, 8] < 1e-4


def test_loss_identities():  # test_renderer.cpp:284-302
    a = np.full((16, 16, 3), 0.2)
    b = np.full((16, 16, 3), 0.7)
    assert orc.loss_value(a, a, 0.2) == 0.0
    assert orc.loss_value(a, b, 0.0) == pytest.approx(0.5, rel=1e-12)
    with pytest.raises(ValueError):
        orc.loss_value(a, np.zeros((15, 16, 3)), 0.2)
    c = random_cloud(10, 80)
    gt = np.full((16, 16, 3), 0.4)
    r = orc.render(c.oracle(), ref_camera(16), cfg())[0]
    expect = np.abs(r - gt).mean() + 0.2 * (1 - orc.ssim(r, gt))
    assert orc.loss_value(r, gt, 0.2) == pytest.approx(expect, rel=1e-12)


def test_backward_forward_matches_render():  # test_renderer.cpp:304-314
    c = random_cloud(12, 81)
    gt = np.full((16, 16, 3), 0.3)
    bw = orc.render_backward(c.oracle(), ref_camera(16), gt, cfg())
    fw = orc.render(c.oracle(), ref_camera(16), cfg())[0]
    assert np.array_equal(bw["rendered"], fw)
    assert bw["loss"] == pytest.approx(orc.loss_value(fw, gt, 0.2), rel=1e-12)
    assert bw["loss"] == pytest.approx(bw["l1"] + 0.2 * (1 - bw["ssim"]), rel=1e-12)


def test_zero_gradients_at_ground_truth():  # test_renderer.cpp:316-332
    c = random_cloud(8, 82)
    gt = orc.render(c.oracle(), ref_camera(16), cfg())[0]
    bw = orc.render_backward(c.oracle(), ref_camera(16), gt, cfg())
    assert bw["loss"] < 1e-12
    for k in ("g_pos", "g_rot", "g_ls", "g_feat", "g_op"):
        assert np.abs(bw[k]).max() < 1e-10


def fd_check(cloud, cam, gt, bw, h=1e-5, tol=1e-3, floor=1e-6):
    rc = cfg()
    worst = 0.0
    for name, gname in (("pos", "g_pos"), ("rot", "g_rot"), ("ls", "g_ls"), ("feat", "g_feat"), ("op", "g_op")):
        arr = getattr(cloud, name)
        for idx in np.ndindex(arr.shape):
            up = cloud.copy(); getattr(up, name)[idx] += h
            dn = cloud.copy(); getattr(dn, name)[idx] -= h
            fu = orc.loss_value(orc.render(up.oracle(), cam, rc)[0], gt, 0.2)
            fdn = orc.loss_value(orc.render(dn.oracle(), cam, rc)[0], gt, 0.2)
            fd = (fu - fdn) / (2 * h)
            g = bw[gname][idx]
            denom = max(abs(fd), abs(g), floor)
            worst = max(worst, abs(fd - g) / denom)
    return worst


def test_analytic_gradients_match_fd():  # test_renderer.cpp:334-371
    c = random_cloud(3, 83)
    cam = ref_camera(12)
    rng = orc.Rng(84)
    gt = np.array([rng.uniform() for _ in range(12 * 12 * 3)]).reshape(12, 12, 3)
    bw = orc.render_backward(c.oracle(), cam, gt, cfg())
    assert fd_check(c, cam, gt, bw) < 1e-3


def test_culled_invisible_zero_grad():  # test_renderer.cpp:373-387
    rows = []
    splat_at(rows, 1, [0, 0, 5], [0.5] * 3, 0.7)
    splat_at(rows, 2, [0, 0, -5], [0.5] * 3, 0.7)
    bw = orc.render_backward(cloud_from_rows(rows).oracle(), axis_camera(100, 8, 17), np.full((17, 17, 3), 0.9), cfg())
    assert bw["visible"][0] == 1 and bw["visible"][1] == 0
    assert bw["screen_grad_norm"][0] > 0 and bw["screen_grad_norm"][1] == 0
    assert np.all(bw["g_pos"][1] == 0) and bw["g_op"][1] == 0 and bw["g_op"][0] != 0


def test_acceptance_crit1_fd_subset():  # acceptance_main.cpp:67-129 (5 of 50 seeds)
    for s in range(5):
        rng = orc.Rng(1000 + s)
        c = grad_check_cloud(rng)
        ex = rng.uniform_range(-0.5, 0.5)  # Vec3(u, u, 5.5): right to left
        ey = rng.uniform_range(-0.5, 0.5)
        cam = orc.look_at([ey, ex, 5.5], [0, 0, 0], [0, 1, 0], 14, 14, 8, 8, 16, 16)
        gt = np.array([rng.uniform() for _ in range(16 * 16 * 3)]).reshape(16, 16, 3)
        bw = orc.render_backward(c.oracle(), cam, gt, cfg())
        # reference re-probes failures at smaller h; abs floor 1e-6
        failed = 0
        for name, gname in (("pos", "g_pos"), ("rot", "g_rot"), ("ls", "g_ls"), ("feat", "g_feat"), ("op", "g_op")):
            arr = getattr(c, name)
            for idx in np.ndindex(arr.shape):
                ok = False
                for h in (1e-5, 1e-6, 1e-7):
                    up = c.copy(); getattr(up, name)[idx] += h
                    dn = c.copy(); getattr(dn, name)[idx] -= h
                    fd = (orc.loss_value(orc.render(up.oracle(), cam, cfg())[0], gt, 0.2) -
                          orc.loss_value(orc.render(dn.oracle(), cam, cfg())[0], gt, 0.2)) / (2 * h)
                    g = bw[gname][idx]
                    err = abs(g - fd)
                    if err <= 1e-6 or err / max(abs(g), abs(fd), 1e-300) <= 1e-3:
                        ok = True
                        break
                failed += not ok
        assert failed == 0


# ---------------------------------------------------------------- test_ssim.cpp
def ssim_direct(x, y):  # test_ssim.cpp:17-51
    w1 = np.array(orc.ssim_window_1d())
    W2 = np.outer(w1, w1)
    H, W, _ = x.shape
    tot, cnt = 0.0, 0
    for ch in range(3):
        for cy in range(5, H - 5):
            for cx in range(5, W - 5):
                a = x[cy - 5:cy + 6, cx - 5:cx + 6, ch]
                b = y[cy - 5:cy + 6, cx - 5:cx + 6, ch]
                mx, my = (W2 * a).sum(), (W2 * b).sum()
                vx = (W2 * a * a).sum() - mx * mx
                vy = (W2 * b * b).sum() - my * my
                cv = (W2 * a * b).sum() - mx * my
                tot += ((2 * mx * my + 1e-4) * (2 * cv + 9e-4)) / ((mx * mx + my * my + 1e-4) * (vx + vy + 9e-4))
                cnt += 1
    return tot / cnt


def test_ssim_window():  # test_ssim.cpp:62-69
    w = orc.ssim_window_1d()
    assert sum(w) == pytest.approx(1.0, rel=1e-12)
    for i in range(5):
        assert w[i] == w[10 - i]
    assert w[5] > w[0]


def test_ssim_identity_and_direct_reference():  # test_ssim.cpp:71-84
    a = random_image(16, 16, 1)
    assert orc.ssim(a, a) == pytest.approx(1.0, rel=1e-12)
    a = random_image(20, 14, 2)
    b = random_image(20, 14, 3)
    assert abs(orc.ssim(a, b) - ssim_direct(a, b)) < 1e-6
    c = 0.7 * a + 0.1
    assert abs(orc.ssim(a, c) - ssim_direct(a, c)) < 1e-6


def test_ssim_closed_form_constants():  # test_ssim.cpp:86-92
    expect = (2 * 0.25 * 0.5 + 1e-4) / (0.25 ** 2 + 0.5 ** 2 + 1e-4)
    assert orc.ssim(np.full((16, 16, 3), 0.25), np.full((16, 16, 3), 0.5)) == pytest.approx(expect, rel=1e-9)


def test_ssim_small_images():  # test_ssim.cpp:94-107
    a, b = random_image(8, 8, 4), random_image(8, 8, 5)
    assert orc.ssim(a, b) == 1.0
    s, dx = orc.ssim_with_gradient(a, b)
    assert s == 1.0 and np.all(dx == 0.0)
    with pytest.raises(ValueError):
        orc.ssim(np.zeros((12, 12, 3)), np.zeros((13, 12, 3)))


def test_ssim_gradient():  # test_ssim.cpp:109-139
    a, b = random_image(16, 12, 6), random_image(16, 12, 7)
    assert orc.ssim_with_gradient(a, b)[0] == pytest.approx(orc.ssim(a, b), rel=1e-12)
    a, b = random_image(13, 13, 8), random_image(13, 13, 9)
    _, dx = orc.ssim_with_gradient(a, b)
    rng = orc.Rng(10)
    h = 1e-6
    for _ in range(24):
        i = rng.uniform_index(a.size)
        ap, am = a.copy().reshape(-1), a.copy().reshape(-1)
        ap[i] += h; am[i] -= h
        fd = (orc.ssim(ap.reshape(a.shape), b) - orc.ssim(am.reshape(a.shape), b)) / (2 * h)
        assert dapprox(dx.reshape(-1)[i], fd, 1e-6)
    a = random_image(14, 14, 11)
    v, dx = orc.ssim_with_gradient(a, a)
    assert v == pytest.approx(1.0, rel=1e-12) and np.abs(dx).max() < 1e-12


# ---------------------------------------------------------------- test_admm.cpp
def rho_only_opacity(v):
    r = orc.Penalties()
    r.rho_p = r.rho_q = r.rho_s = r.rho_f = 0.0
    r.rho_o = v
    return r


def test_scalar_penalty_example():  # test_admm.cpp:71-88
    x, z, u = scalar_cloud(7, 3.0), scalar_cloud(7, 1.0), scalar_cloud(7, 0.5)
    d = orc.penalty_loss_and_grad(x.oracle(), [0], z.oracle(), u.oracle(), rho_only_opacity(2.0))
    assert d["loss"] == pytest.approx(6.25, rel=1e-15)
    assert d["g_op"][0] == pytest.approx(5.0, rel=1e-15)
    assert np.all(d["g_pos"] == 0)


def test_penalty_zero_at_consensus_and_misaligned():  # test_admm.cpp:90-120
    x = random_bundle([1, 2, 3], 5)
    u = orc.zero_bundle([1, 2, 3], 3)
    d = orc.penalty_loss_and_grad(x.oracle(), [0, 1, 2], x.oracle(), u, orc.Penalties())
    assert d["loss"] == 0.0 and np.all(d["g_pos"] == 0) and np.all(d["g_rot"] == 0)
    with pytest.raises(ValueError):
        orc.penalty_loss_and_grad(scalar_cloud(1, 2.0).oracle(), [0], scalar_cloud(2, 0.0).oracle(),
                                  scalar_cloud(1, 0.0).oracle(), orc.Penalties())


def test_consensus_examples():  # test_admm.cpp:196-266
    a = random_bundle([1, 5, 9], 20)
    z, _ = orc.consensus_average([(0, a.oracle()), (1, a.oracle())], False, empty_cloud().oracle(), 1.0)
    assert z.checksum() == a.oracle().checksum()
    z, _ = orc.consensus_average([(0, scalar_cloud(4, 1.0).oracle()), (1, scalar_cloud(4, 3.0).oracle())], False,
                                 empty_cloud().oracle(), 1.0)
    assert z.dict()["op"][0] == pytest.approx(2.0, rel=1e-15)
    # sign alignment (test_admm.cpp:233-248)
    qa = np.array([0.9, 0.1, 0.2, 0.3]); qa /= np.linalg.norm(qa)
    A, B = scalar_cloud(1, 0.0), scalar_cloud(1, 0.0)
    A.rot[0] = qa; B.rot[0] = -qa
    z, flipped = orc.consensus_average([(0, A.oracle()), (1, B.oracle())], False, empty_cloud().oracle(), 1.0)
    assert np.abs(z.dict()["rot"][0] - qa).max() < 1e-15 and flipped == [1]
    # not renormalized (test_admm.cpp:250-259)
    A.rot[0] = [1, 0, 0, 0]; B.rot[0] = [0, 1, 0, 0]
    z, _ = orc.consensus_average([(0, A.oracle()), (1, B.oracle())], False, empty_cloud().oracle(), 1.0)
    assert list(z.dict()["rot"][0]) == [0.5, 0.5, 0, 0]
    # over-relaxation (test_admm.cpp:261-276)
    z, _ = orc.consensus_average([(0, scalar_cloud(1, 2.0).oracle()), (1, scalar_cloud(1, 4.0).oracle())], True,
                                 scalar_cloud(1, 1.0).oracle(), 1.6)
    assert z.dict()["op"][0] == pytest.approx(0.5 * ((1.6 * 2 - 0.6) + (1.6 * 4 - 0.6)), rel=1e-15)
    z2, _ = orc.consensus_average([(0, scalar_cloud(9, 3.0).oracle())], True, scalar_cloud(1, 1.0).oracle(), 1.6)
    assert z2.dict()["op"][0] == 3.0


def test_dual_update_and_residuals():  # test_admm.cpp:278-320
    u = orc.dual_update(scalar_cloud(1, 0.5).oracle(), scalar_cloud(1, 3.0).oracle(), scalar_cloud(1, 1.0).oracle())
    assert u.dict()["op"][0] == pytest.approx(2.5, rel=1e-15)
    with pytest.raises(ValueError):
        orc.dual_update(scalar_cloud(1, 0.5).oracle(), scalar_cloud(2, 3.0).oracle(), scalar_cloud(1, 1.0).oracle())
    r = orc.Penalties(); r.rho_p = r.rho_q = r.rho_s = r.rho_f = r.rho_o = 4.0
    p, d = orc.residuals([(0, scalar_cloud(1, 2.0).oracle())], scalar_cloud(1, 1.0).oracle(), scalar_cloud(1, 1.0).oracle(), r)
    assert p == pytest.approx(1.0, rel=1e-15) and d == 0.0


def test_adapt_penalties():  # test_admm.cpp:322-355
    cc = orc.ConsensusConfig()
    rho = orc.Penalties()
    assert orc.adapt_penalties(rho, 2.0, 0.1, cc, 100).rho_p == pytest.approx(2e4)
    assert orc.adapt_penalties(rho, 0.1, 2.0, cc, 100).rho_f == pytest.approx(5e2)
    assert orc.adapt_penalties(rho, 1.0, 1.0, cc, 100).rho_p == rho.rho_p
    assert orc.adapt_penalties(rho, 2.0, 0.1, cc, cc.freeze_iteration + 1).rho_p == rho.rho_p


def test_max_disagreement():  # test_admm.cpp:357-368
    a, b, c = scalar_cloud(1, 0.0), scalar_cloud(1, 0.0), scalar_cloud(2, 99.0)
    b.pos[0] = [0.25, 0, 0]
    assert orc.max_disagreement([(0, a.oracle()), (1, b.oracle()), (2, c.oracle())]) == pytest.approx(0.25, rel=1e-15)
    assert orc.max_disagreement([(0, a.oracle()), (1, a.oracle())]) == 0.0


# ------------------------------------------------------------- test_trainer.cpp
def spread_cloud(n, log_scale, opacity0=0.5):  # test_trainer.cpp:48-60
    rows = [(i, [i * 5.0 - 2.5 * (n - 1), 0, 5], [1.0, 0, 0, 0], [log_scale] * 3, [1.5, 1.0, 0.5],
             logit(opacity0 if i == 0 else 0.5)) for i in range(n)]
    return cloud_from_rows(rows)


def quiet(iters):
    tc = orc.TrainerConfig()
    tc.iterations = iters
    tc.densify_enabled = False
    return tc


def test_trainer_deterministic():  # test_trainer.cpp:172-183
    c = spread_cloud(3, -1.5)
    cam = orc.look_at([0, 1, -4], [0, 0, 5], [0, 1, 0], 12, 12, 6, 6, 12, 12)
    gt = np.full((12, 12, 3), 0.4)
    tc = quiet(100)
    tc.seed = 7
    a = orc.BlockTrainer(0, c.oracle(), [cam], [gt], [], 3, tc)
    b = orc.BlockTrainer(0, c.oracle(), [cam], [gt], [], 3, tc)
    a.run_iterations(30); b.run_iterations(30)
    assert a.cloud().checksum() == b.cloud().checksum() and a.last_loss() == b.last_loss()


def test_trainer_descends_on_toy_scene():  # test_trainer.cpp:136-170
    sc = orc.SynthConfig()
    sc.seed, sc.gaussians, sc.cameras, sc.image_size, sc.extent = 3, 12, 4, 24, 4.0
    s = orc.generate_scene(sc)
    tc = orc.TrainerConfig()
    tc.iterations, tc.seed, tc.densify_interval = 150, 1, 60
    p, c = s.points()  # positions f32, rgb u8
    init = orc.init_cloud_from_points(p, c, 0, tc.init_opacity)
    ims = s.images()
    mean_loss = lambda cl: np.mean([orc.loss_value(orc.render(cl, v, tc.render)[0], im, 0.2) for v, im in zip(s.views, ims)])
    before = mean_loss(init)
    t = orc.BlockTrainer(0, init, s.views, ims, [], init.size(), tc)
    t.run_iterations(150)
    assert mean_loss(t.cloud()) < 0.7 * before
    assert t.last_loss() > 0 and t.iteration() == 150


def test_anchor_and_broadcast():  # test_trainer.cpp:275-306
    c = spread_cloud(3, -2.0)
    cam = orc.look_at([0, 0, -5], [0, 0, 5], [0, 1, 0], 10, 10, 4, 4, 8, 8)
    t = orc.BlockTrainer(0, c.oracle(), [cam], [np.zeros((8, 8, 3))], [0, 1], 3, quiet(100))
    rho = orc.Penalties()
    z0 = HostCloud.from_oracle(orc.slice_by_ids(c.oracle(), [0, 1]))
    z0.op += 0.25
    t.set_anchor(z0.oracle(), rho)
    assert list(t.anchor().dict()["ids"]) == [0, 1] and np.all(t.duals().dict()["op"] == 0)
    z1 = HostCloud.from_oracle(orc.slice_by_ids(c.oracle(), [0]))
    z1.op -= 0.5
    t.apply_broadcast(z1.oracle(), [], [1], rho, 1.0, False)
    assert t.shared_ids() == [0]
    assert t.duals().dict()["op"][0] == pytest.approx(0.5, rel=1e-12)
    assert np.all(t.duals().dict()["pos"][0] == 0)
    t.apply_broadcast(z1.oracle(), [0], [], rho, 1.0, False)
    assert t.duals().dict()["op"][0] == 0.0


def test_penalty_pulls_invisible_gaussian():  # test_trainer.cpp:308-338
    c = cloud_from_rows([(0, [0, 0, -10], [1.0, 0, 0, 0], [-1] * 3, [1, 1, 1], 2.0)])
    cam = orc.look_at([0, 0, 20], [0, 0, 25], [0, 1, 0], 10, 10, 4, 4, 8, 8)
    t = orc.BlockTrainer(0, c.oracle(), [cam], [np.zeros((8, 8, 3))], [0], 1, quiet(100))
    z = c.copy(); z.op[0] = -1.0; z.pos[0, 0] = 1.0
    t.set_anchor(z.oracle(), orc.Penalties())
    t.run_iterations(10)
    d = t.cloud().dict()
    assert abs(d["op"][0] - (-1.0)) < abs(2.0 - (-1.0))
    assert abs(d["pos"][0, 0] - 1.0) < 1.0


# ------------------------------------------------------------ test_splitter.cpp
def test_splitter_balanced_and_vertical_never_split():  # test_splitter.cpp (50/50, vertical axis)
    rng = np.random.default_rng(0)
    pts = np.stack([rng.uniform(-10, 10, 1000), rng.uniform(-100, 100, 1000), rng.uniform(-5, 5, 1000)], 1)
    g = HostCloud(np.arange(1000, dtype=np.uint64), pts, np.tile([1.0, 0, 0, 0], (1000, 1)), np.zeros((1000, 3)),
                  np.zeros((1000, 3)), np.zeros(1000))
    d = orc.split_and_assign(pts, 2, [], g.oracle(), 1.0, 1, False)
    assert [len(c) for c in d["core_points"]] == [500, 500]
    # x is the longer ground axis; the tall y axis is never split
    assert d["core_max"][0][0] <= d["core_min"][1][0]
    d8 = orc.split_and_assign(pts, 8, [], g.oracle(), 1.4, 1, False)
    sizes = [len(c) for c in d8["core_points"]]
    assert max(sizes) - min(sizes) <= 1
    # expanded boxes contain the core boxes and span the full vertical range
    assert np.all(d8["exp_min"] <= d8["core_min"]) and np.all(d8["exp_max"] >= d8["core_max"])
    assert np.all(d8["exp_min"][:, 1] == pts[:, 1].min())
    # every gaussian is owned; shared ids have >= 2 owners, ascending
    owned = set()
    for b in d8["block_gaussians"]:
        owned |= set(b)
    assert owned == set(range(1000))
    for gid, who in d8["shared"].items():
        assert len(who) >= 2 and who == sorted(who)


def test_consensus_schedule():  # runtime.cpp:256-263
    assert orc.consensus_schedule(100, 10) == list(range(10, 101, 10))
    assert orc.consensus_schedule(25, 10) == [10, 20, 25]
