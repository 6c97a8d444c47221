"""GPU parity of the training step (fused fold + ADMM penalty + Adam,
trainer.cpp:249-295) and of the consensus round (admm.cpp:71-198,
trainer.cpp:168-223) against the oracle, through the C-ABI."""
import numpy as np
import pytest

import _oracle as orc
from gpu_helpers import check_adam_trajectory, dev_cam, gpu, new_block
from paper_2405_13943_b200 import api
from refcases import HostCloud, random_bundle

pytestmark = gpu


def toy_scene(seed=3, gaussians=40, cameras=6, size=32, extent=4.0):
    sc = orc.SynthConfig()
    sc.seed, sc.gaussians, sc.cameras, sc.image_size, sc.extent = seed, gaussians, cameras, size, extent
    s = orc.generate_scene(sc)
    p, c = s.points()
    init = HostCloud.from_oracle(orc.init_cloud_from_points(p, c, 0, 0.1)).narrowed()
    return s, init


def oracle_cfg(iters, seed=1):
    tc = orc.TrainerConfig()
    tc.iterations, tc.seed = iters, seed
    tc.densify_enabled = False
    return tc


def device_trainer(init, s):
    b = new_block(init)
    b.set_views([dev_cam(v) for v in s.views], s.images())
    b.trainer_init(api.trainer_config(iterations=20))
    return b


def rows_of(hc):
    return np.concatenate([hc.pos, hc.rot, hc.ls, hc.feat, hc.op[:, None]], 1)


@pytest.mark.parametrize("steps", [1, 10])
def test_train_steps_track_oracle(steps):
    s, init = toy_scene()
    tc = oracle_cfg(20)
    t = orc.BlockTrainer(0, init.oracle(), s.views, s.images(), [], init.n, tc)
    seq = orc.view_sequence(1, 0, len(s.views), steps)
    b = device_trainer(init, s)
    losses = b.train_steps(seq)
    images = s.images()
    grads, want_losses = [], []
    for k in range(steps):
        grads.append(orc.render_backward(t.cloud(), s.views[seq[k]], images[seq[k]], orc.RenderConfig()))
        want_losses.append(t.train_step())
    np.testing.assert_allclose(losses, want_losses, rtol=2e-4)
    got = b.download_cloud()
    check_adam_trajectory(got, t.cloud().dict(), grads, api.trainer_config(iterations=20), steps)
    m, v = b.moments()
    assert np.all(np.isfinite(m)) and np.all(v >= 0)
    ga, gs = b.densify_stats()
    assert np.array_equal(gs, np.array(t.grad_seen(), dtype=np.uint32))
    np.testing.assert_allclose(ga, t.grad_accum(), rtol=5e-3, atol=1e-9)


def test_penalty_pulls_invisible_gaussian_on_device():
    """test_trainer.cpp:308-338 through the fused kernel."""
    c = HostCloud(np.array([0], np.uint64), [[0, 0, -10]], [[1.0, 0, 0, 0]], [[-1, -1, -1]], [[1, 1, 1]], [2.0])
    cam = orc.look_at([0, 0, 20], [0, 0, 25], [0, 1, 0], 10, 10, 4, 4, 8, 8)
    b = new_block(c)
    b.set_views([dev_cam(cam)], [np.zeros((8, 8, 3))])
    b.trainer_init(api.trainer_config(iterations=100))
    b.set_shared([0], [0], [1], [1])
    z = np.concatenate([c.pos, c.rot, c.ls, c.feat, c.op[:, None]], 1).copy()
    z[0, 13] = -1.0
    z[0, 0] = 1.0
    b.set_anchor(z, z, api.penalties())
    b.train_steps([0] * 10)
    got = b.download_cloud()
    assert abs(got["op"][0] - (-1.0)) < 3.0
    assert abs(got["pos"][0, 0] - 1.0) < 1.0
    t = orc.BlockTrainer(0, c.oracle(), [cam], [np.zeros((8, 8, 3))], [0], 1, oracle_cfg(100))
    zc = c.copy(); zc.op[0] = -1.0; zc.pos[0, 0] = 1.0
    t.set_anchor(zc.oracle(), orc.Penalties())
    t.run_iterations(10)
    want = t.cloud().dict()
    np.testing.assert_allclose(got["op"], want["op"], atol=1e-4)
    np.testing.assert_allclose(got["pos"], want["pos"], atol=1e-4)


def _sh1(hc, seed):
    g = np.random.default_rng(seed)
    feat = np.concatenate([hc.feat[:, :3], 0.3 * g.standard_normal((hc.n, 9))], 1)
    return HostCloud(hc.ids, hc.pos, hc.rot, hc.ls, feat, hc.op)


def make_blocks_for_consensus(flip_ids=(3,), fd=3):
    """Two blocks sharing ids {2..7} (block 0 owns 0..7, block 1 owns 2..11)."""
    a = random_bundle(list(range(0, 8)), 40)
    b = random_bundle(list(range(2, 12)), 41)
    if fd == 12:
        a, b = _sh1(a, 1), _sh1(b, 2)
    a, b = a.narrowed(), b.narrowed()
    # shared rows of block 1 close to block 0's, with one antipodal quaternion
    for gid in range(2, 8):
        ia, ib = gid, gid - 2
        b.pos[ib] = a.pos[ia] + 0.01 * (gid % 3)
        b.rot[ib] = a.rot[ia] * (-1.0 if gid in flip_ids else 1.0)
    b = b.narrowed()
    shared = list(range(2, 8))
    zprev = random_bundle(shared, 42)
    zprev = (_sh1(zprev, 3) if fd == 12 else zprev).narrowed()
    return a, b, shared, zprev


def setup_device_block(hc, shared, block_id, zprev, rho):
    dev = new_block(hc)
    rows = [int(np.searchsorted(hc.ids, g)) for g in shared]
    slots = list(range(len(shared)))
    first = [1 if block_id == 0 else 0] * len(shared)
    dev.set_shared(rows, slots, first, [2] * len(shared))
    zp = rows_of(zprev)
    dev.set_anchor(zp, zp, rho)
    return dev


@pytest.mark.parametrize("relax,fd", [(False, 3), (True, 3), (True, 12)])
def test_consensus_round_matches_oracle(relax, fd):
    a, b, shared, zprev = make_blocks_for_consensus(fd=fd)
    rho = api.penalties()
    da = setup_device_block(a, shared, 0, zprev, rho)
    db = setup_device_block(b, shared, 1, zprev, rho)
    alpha = 1.6
    res = api.group_consensus_round([da, db], alpha, relax, diagnostics=True)
    sa = orc.slice_by_ids(a.oracle(), shared)
    sb = orc.slice_by_ids(b.oracle(), shared)
    z, flipped = orc.consensus_average([(0, sa), (1, sb)], relax, zprev.oracle(), alpha)
    zr = rows_of(HostCloud.from_oracle(z))
    np.testing.assert_allclose(da.consensus(), zr, rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(db.consensus(), zr, rtol=1e-6, atol=1e-6)
    assert res["flipped"] == len(flipped) == 1
    p, d = orc.residuals([(0, sa), (1, sb)], z, zprev.oracle(), orc.Penalties())
    assert res["primal"] == pytest.approx(p, rel=1e-5)
    assert res["dual"] == pytest.approx(d, rel=1e-4)
    # duals: u = 0 + x_hat - z (x_hat relaxed against the anchor, no flip), flipped ids reset
    for dev, hc in ((da, a), (db, b)):
        x = rows_of(HostCloud.from_oracle(orc.slice_by_ids(hc.oracle(), shared)))
        xh = alpha * x + (1 - alpha) * rows_of(zprev) if relax else x
        want_u = xh - zr
        for k, gid in enumerate(shared):
            if gid in flipped:
                want_u[k] = 0
        np.testing.assert_allclose(dev.duals(), want_u, rtol=1e-5, atol=2e-6)
        np.testing.assert_allclose(dev.anchor(), zr, rtol=1e-6, atol=1e-6)
    # dual-mean diagnostic (runtime.cpp:572-606) and disagreement (admm.cpp:219-243)
    assert res["max_disagreement"] == pytest.approx(orc.max_disagreement([(0, sa), (1, sb)]), rel=1e-5)


def _anchored_trainer(init, s, shared_rows, zprev_rows, rho):
    b = device_trainer(init, s)
    n = len(shared_rows)
    b.set_shared(shared_rows, list(range(n)), [1] * n, [1] * n)
    b.set_anchor(zprev_rows, zprev_rows, rho)
    return b


def test_async_round_overlaps_next_step_exactly():
    """an asynchronous round (comm stream, device-side penalty
    adaptation) followed immediately by train steps -- whose Adam waits for the
    round -- equals a synchronous round, host-side adapt_penalties
    (admm.cpp:200-217) and the same steps."""
    s, init = toy_scene()
    shared_rows = list(range(0, init.n, 3))
    g = np.random.default_rng(5)
    x0 = rows_of(init)[shared_rows]
    zprev = (x0 + 0.05 * g.standard_normal(x0.shape)).astype(np.float32).astype(np.float64)
    rho = api.penalties()
    seq = orc.view_sequence(1, 0, len(s.views), 12)
    # synchronous reference
    a = _anchored_trainer(init, s, shared_rows, zprev, rho)
    a.train_steps(seq[:4])
    ra = a.consensus_round(1.6, True)
    mu, tau_inc, tau_dec = 10.0, 2.0, 2.0
    f = 1.0
    if ra["primal"] > mu * ra["dual"]:
        f = tau_inc
    elif ra["dual"] > mu * ra["primal"]:
        f = 1.0 / tau_dec
    rho_a = api.penalties(**{k: getattr(rho, k) * f for k in ("rho_p", "rho_q", "rho_s", "rho_f", "rho_o")})
    a.set_penalties(rho_a)
    la = a.train_steps(seq[4:12])
    # asynchronous: the round is in flight while the next steps project/sort/blend
    b = _anchored_trainer(init, s, shared_rows, zprev, rho)
    b.train_steps(seq[:4])
    b.consensus_round_async(1.6, True, iteration=4, mu=mu, tau_inc=tau_inc, tau_dec=tau_dec)
    lb = b.train_steps(seq[4:12])
    rb = b.consensus_wait()
    assert f != 1.0  # the case exercises the adaptation
    assert rb["rho"] == pytest.approx((rho_a.rho_p, rho_a.rho_q, rho_a.rho_s, rho_a.rho_f, rho_a.rho_o), rel=1e-12)
    assert rb["primal"] == pytest.approx(ra["primal"], rel=1e-6)
    assert rb["dual"] == pytest.approx(ra["dual"], rel=1e-6)
    np.testing.assert_allclose(lb, la, rtol=1e-4)
    np.testing.assert_allclose(b.duals(), a.duals(), rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(b.anchor(), a.anchor(), rtol=1e-5, atol=1e-6)
    # The two runs differ only by the order of the blend backward's FP32
    # atomics (the gradients agree to ~1e-7 relative); Adam turns that into
    # differences of up to 2 lr per step on coordinates whose gradient is
    # near zero, so: every coordinate within that bound, all but 1% (at
    # least 2) within 1e-5.
    ga, gb = a.download_cloud(), b.download_cloud()
    lr = {"pos": 1.6e-4, "rot": 1e-3, "ls": 5e-3, "feat": 2.5e-3, "op": 5e-2}
    for k in ("pos", "rot", "ls", "feat", "op"):
        err = np.abs(gb[k] - ga[k])
        assert np.all(err <= 2 * lr[k] * 8 + 1e-6), (k, err.max())
        far = int(np.sum(err > 1e-5 + 1e-4 * np.abs(ga[k])))
        assert far <= max(2, err.size // 100), (k, far)


def test_async_round_then_densify_waits_for_the_round():
    """An asynchronous round still pending when the next bsg_train_steps crosses
    a densification iteration (bsg_consensus_round_async, then train steps):
    densification waits for the round (it rewrites the anchor / dual rows the
    round writes) and the round's result stays pending for consensus_wait.
    Same densify decisions, round result and trajectory as the synchronous
    order (round, wait, then the steps)."""
    s, init = toy_scene(gaussians=120, cameras=6, size=40)
    shared_rows = list(range(0, init.n, 4))
    x0 = rows_of(init)[shared_rows]
    zprev = (x0 + 0.02 * np.random.default_rng(6).standard_normal(x0.shape)).astype(np.float32).astype(np.float64)
    rho = api.penalties()
    seq = orc.view_sequence(1, 0, len(s.views), 10)
    # densify at iteration 6 with thresholds that act on this scene: a probe run places them
    probe = _anchored_trainer(init, s, shared_rows, zprev, rho)
    probe.train_steps(seq[:6])
    ga, gs = probe.densify_stats()
    pc = probe.download_cloud()
    grad_thr = _midpoint_threshold(ga[gs > 0] / gs[gs > 0], 0.5)
    prune = _midpoint_threshold(1 / (1 + np.exp(-pc["op"])), 0.2)
    dens = dict(enabled=1, interval=6, stop_iteration=6, grad_threshold=grad_thr, prune_opacity=prune,
                split_scale_fraction=0.01, split_shrink=1.6)

    def trainer():
        b = new_block(init)
        b.set_views([dev_cam(v) for v in s.views], s.images())
        b.trainer_init(api.trainer_config(iterations=20, densify=dens))
        n = len(shared_rows)
        b.set_shared(shared_rows, list(range(n)), [1] * n, [1] * n)
        b.set_anchor(zprev, zprev, rho)
        return b

    a = trainer()
    a.train_steps(seq[:4])
    ra = a.consensus_round(1.6, True)
    la = a.train_steps(seq[4:10])
    b = trainer()
    b.train_steps(seq[:4])
    b.consensus_round_async(1.6, True)
    lb = b.train_steps(seq[4:10])  # iteration 6 densifies while the round may be in flight
    rb = b.consensus_wait()
    assert rb["primal"] == pytest.approx(ra["primal"], rel=1e-6)
    assert rb["dual"] == pytest.approx(ra["dual"], rel=1e-6)
    removed_a, removed_b = list(a.take_removed_ids()), list(b.take_removed_ids())
    assert len(removed_a) > 0 and removed_a == removed_b
    assert np.array_equal(a.take_new_ids(), b.take_new_ids())
    assert list(a.shared_ids()) == list(b.shared_ids())
    np.testing.assert_allclose(lb, la, rtol=1e-4)
    ga_, gb_ = a.download_cloud(), b.download_cloud()
    assert np.array_equal(ga_["ids"], gb_["ids"])
    np.testing.assert_allclose(gb_["pos"], ga_["pos"], rtol=1e-4, atol=1e-5)


def test_evaluate_matches_reference_metrics():
    """evaluate (metrics.cpp:28-51) on the device: holdout rule, PSNR
    (metrics.cpp:14-26) and SSIM (ssim.cpp) vs the FP64 oracle rendering."""
    s, init = toy_scene(size=40)
    ims = s.images()
    b = new_block(init)
    for holdout in (3, 0):
        got = b.evaluate([dev_cam(v) for v in s.views], ims, holdout_modulus=holdout)
        idx = [i for i in range(len(s.views)) if holdout == 0 or i % holdout == 0]
        assert len(got["psnr"]) == len(idx)
        for k, i in enumerate(idx):
            r = orc.render(init.oracle(), s.views[i], orc.RenderConfig())[0]
            assert got["psnr"][k] == pytest.approx(orc.psnr(r, ims[i]), abs=1e-4)
            assert got["ssim"][k] == pytest.approx(orc.ssim(r, ims[i]), abs=1e-5)
        assert got["mean_psnr"] == pytest.approx(np.mean(got["psnr"]), rel=1e-12)
    # identical images are capped at 99 dB
    r0 = orc.render(init.oracle(), s.views[0], orc.RenderConfig())[0]
    capped = b.evaluate([dev_cam(s.views[0])], [b.render(dev_cam(s.views[0]))[0]], holdout_modulus=0)
    assert capped["psnr"][0] == 99.0 and capped["ssim"][0] == pytest.approx(1.0, abs=1e-6)
    assert np.abs(b.render(dev_cam(s.views[0]))[0] - r0).max() < 1e-4
    assert len(b.evaluate([dev_cam(s.views[1])], [ims[1]], holdout_modulus=2)["psnr"]) == 1  # index 0 qualifies
    with pytest.raises(api.InvalidArgument):
        b.evaluate([], [], holdout_modulus=1)  # metrics.cpp:44 "empty holdout"


def _midpoint_threshold(values, q):
    """A threshold between two neighbouring sorted values near quantile q, so
    FP32-vs-FP64 differences cannot flip a decision."""
    v = np.sort(np.asarray(values, np.float64))
    k = int(np.clip(round(q * (len(v) - 1)), 1, len(v) - 1))
    gaps = np.diff(v)
    lo = max(1, k - 3)
    j = lo + int(np.argmax(gaps[lo - 1:k + 3]))  # widest gap near the quantile
    return 0.5 * (v[j - 1] + v[j])


@pytest.mark.parametrize("shared_every", [0, 4])
def test_densify_matches_oracle(shared_every):
    """maybe_densify (trainer.cpp:301-385) on the device: prune / clone / split
    (non-shared) / bud (shared) decisions, block-disjoint ids, optimizer state
    compaction and the shared-set shrink, against the oracle trainer."""
    s, init = toy_scene(gaussians=120, cameras=6, size=40)
    steps = 6
    shared = [int(i) for i in init.ids[::shared_every]] if shared_every else []
    rows = [int(np.searchsorted(init.ids, g)) for g in shared]
    anchor = HostCloud(init.ids[rows], init.pos[rows], init.rot[rows], init.ls[rows], init.feat[rows], init.op[rows])

    def oracle_trainer(tc):
        t = orc.BlockTrainer(0, init.oracle(), s.views, s.images(), shared, init.n, tc)
        if shared:
            t.set_anchor(anchor.oracle(), orc.Penalties())
        return t

    # probe the state at the densification point to place every threshold in a gap
    probe = oracle_trainer(oracle_cfg(30))
    for _ in range(steps):
        probe.train_step()
    ga, gs = np.array(probe.grad_accum()), np.array(probe.grad_seen())
    pc = HostCloud.from_oracle(probe.cloud())
    grad_thr = _midpoint_threshold(ga[gs > 0] / gs[gs > 0], 0.5)
    prune = _midpoint_threshold(1 / (1 + np.exp(-pc.op)), 0.2)
    lo, hi = init.pos.min(0), init.pos.max(0)
    extent = np.sqrt(((hi - lo) ** 2).sum())
    frac = _midpoint_threshold(np.exp(pc.ls).max(1) / extent, 0.5)
    dens = dict(enabled=1, interval=steps, stop_iteration=steps, grad_threshold=grad_thr, prune_opacity=prune,
                split_scale_fraction=frac, split_shrink=1.6)
    tc = oracle_cfg(30)
    tc.densify_enabled, tc.densify_interval, tc.densify_stop_iteration = True, steps, steps
    tc.densify_grad_threshold, tc.densify_prune_opacity, tc.densify_split_scale_fraction = grad_thr, prune, frac
    t = oracle_trainer(tc)
    n_steps = steps + 3
    want_losses = [t.train_step() for _ in range(n_steps)]
    b = new_block(init)
    b.set_views([dev_cam(v) for v in s.views], s.images())
    b.trainer_init(api.trainer_config(iterations=30, densify=dens))
    if shared:
        b.set_shared(rows, list(range(len(rows))), [1] * len(rows), [1] * len(rows))
        z = rows_of(anchor)
        b.set_anchor(z, z, api.penalties())
    seq = orc.view_sequence(1, 0, len(s.views), n_steps)
    losses = b.train_steps(seq)
    want = HostCloud.from_oracle(t.cloud())
    got = b.download_cloud()
    # the decisions are integer: same ids in the same rows
    removed, new = list(t.take_removed_ids()), HostCloud.from_oracle(t.take_new_rows()).ids
    assert len(removed) > 0 and len(new) > 0
    assert np.array_equal(got["ids"], want.ids)
    assert list(b.take_removed_ids()) == removed
    assert np.array_equal(b.take_new_ids(), new)
    assert all(int(i) >= init.n for i in new)  # block 0 allocates past the initial ids
    if shared:
        assert list(b.shared_ids()) == list(t.shared_ids())
    # before the densification the trajectories agree to FP32 rounding; after it
    # the children start from FP32 vs FP64 parents (one view's small loss moved 0.7%)
    np.testing.assert_allclose(losses[:steps], want_losses[:steps], rtol=5e-4)
    np.testing.assert_allclose(losses[steps:], want_losses[steps:], rtol=1e-2)
    g = np.concatenate([got["pos"], got["rot"], got["ls"], got["feat"], got["op"][:, None]], 1)
    err = np.abs(g - rows_of(want))
    assert np.mean(err <= 1e-4 + 1e-4 * np.abs(rows_of(want))) >= 0.98
    m, v = b.moments()
    assert m.shape[1] == len(want.ids) and np.all(v >= 0)


def test_nccl_round_path_single_rank():
    """The NCCL code path of the round (dlopen'd libnccl, AllReduces on the
    communication stream) with a one-rank communicator: same result as the
    communicator-less round."""
    s, init = toy_scene()
    shared_rows = list(range(0, init.n, 2))
    x0 = rows_of(init)[shared_rows]
    zprev = (x0 + 0.02).astype(np.float32).astype(np.float64)
    seq = orc.view_sequence(1, 0, len(s.views), 6)
    out = []
    for use_nccl in (False, True):
        b = _anchored_trainer(init, s, shared_rows, zprev, api.penalties())
        if use_nccl:
            b.comm_init(api.nccl_unique_id(), 1, 0)
        b.train_steps(seq[:3])
        b.consensus_round_async(1.6, True, iteration=3)
        b.train_steps(seq[3:])
        r = b.consensus_wait()
        out.append((r, b.anchor(), b.duals()))
    (ra, za, ua), (rb, zb, ub) = out
    assert rb["primal"] == pytest.approx(ra["primal"], rel=1e-6)
    assert rb["dual"] == pytest.approx(ra["dual"], rel=1e-6)
    assert rb["rho"] == ra["rho"]
    np.testing.assert_allclose(zb, za, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(ub, ua, rtol=1e-5, atol=1e-6)


def test_sh1_train_steps_track_oracle():
    """Adam and the fold over D = 23 components (SH degree 1)."""
    s, init = toy_scene()
    g = np.random.default_rng(7)
    feat = np.concatenate([init.feat[:, :3], 0.3 * g.standard_normal((init.n, 9))], 1)
    init = HostCloud(init.ids, init.pos, init.rot, init.ls, feat, init.op).narrowed()
    tc = oracle_cfg(20)
    t = orc.BlockTrainer(0, init.oracle(), s.views, s.images(), [], init.n, tc)
    seq = orc.view_sequence(1, 0, len(s.views), 6)
    b = device_trainer(init, s)
    losses = b.train_steps(seq)
    want_losses = [t.train_step() for _ in range(6)]
    np.testing.assert_allclose(losses, want_losses, rtol=2e-4)
    got = b.download_cloud()
    want = HostCloud.from_oracle(t.cloud())
    gr = np.concatenate([got["pos"], got["rot"], got["ls"], got["feat"], got["op"][:, None]], 1)
    err = np.abs(gr - rows_of(want))
    assert np.mean(err <= 1e-5 + 1e-5 * np.abs(rows_of(want))) >= 0.98


@pytest.mark.parametrize("case", ["nothing-visible", "tiny-image", "empty-cloud"])
def test_train_step_edge_cases_track_oracle(case):
    """Steps where the raster has nothing to do (every splat culled; V = P = 0),
    an image smaller than the SSIM window (ssim.cpp:12-14: SSIM = 1, zero
    gradient), and an empty cloud: loss and the dense Adam (moments decay,
    invisible rows move, trainer.cpp:267-281) still match the oracle."""
    s, init = toy_scene()
    views, imgs = list(s.views), s.images()
    if case == "nothing-visible":
        cam = orc.look_at([0.0, 0.0, 50.0], [0.0, 0.0, 100.0], [0.0, 1.0, 0.0], 30, 30, 16, 16, 32, 32)
        views, imgs = [cam], [np.full((32, 32, 3), 0.25)]
    elif case == "tiny-image":
        cam = orc.look_at([0.0, 0.5, -6.0], [0.0, 0.0, 0.0], [0.0, 1.0, 0.0], 8, 8, 4, 4, 8, 8)
        views, imgs = [cam], [np.full((8, 8, 3), 0.4)]
    else:
        init = HostCloud(np.zeros(0, np.uint64), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)),
                         np.zeros((0, 3)), np.zeros(0))
        views, imgs = views[:2], imgs[:2]
    t = orc.BlockTrainer(0, init.oracle(), views, imgs, [], max(init.n, 1), oracle_cfg(20))
    b = new_block(init)
    b.set_views([dev_cam(v) for v in views], imgs)
    b.trainer_init(api.trainer_config(iterations=20))
    seq = orc.view_sequence(1, 0, len(views), 4)
    losses = b.train_steps(seq)
    want = [t.train_step() for _ in range(4)]
    np.testing.assert_allclose(losses, want, rtol=2e-4, atol=1e-9)
    if init.n:
        got = b.download_cloud()
        w = HostCloud.from_oracle(t.cloud())
        g = np.concatenate([got["pos"], got["rot"], got["ls"], got["feat"], got["op"][:, None]], 1)
        assert np.mean(np.abs(g - rows_of(w)) <= 1e-5 + 1e-5 * np.abs(rows_of(w))) >= 0.98


def test_train_steps_host_matches_resident_views():
    """bsg_train_steps_host (host images, double-buffered uploads) trains like
    bsg_train_steps on the same views resident on the device."""
    s, init = toy_scene(seed=5)
    seq = orc.view_sequence(1, 0, len(s.views), 9)
    a = device_trainer(init, s)
    la = a.train_steps(seq)
    b = device_trainer(init, s)
    ims = s.images()
    cams = [dev_cam(s.views[v]) for v in seq]
    lb = b.train_steps_host(cams, [np.ascontiguousarray(ims[v], dtype=np.float32) for v in seq])
    np.testing.assert_allclose(lb, la, rtol=1e-5)
    ca, cb = a.download_cloud(), b.download_cloud()
    ga = np.concatenate([ca["pos"], ca["rot"], ca["ls"], ca["feat"], ca["op"][:, None]], 1)
    gb = np.concatenate([cb["pos"], cb["rot"], cb["ls"], cb["feat"], cb["op"][:, None]], 1)
    # both runs reduce gradients with float atomics (order not fixed): Adam
    # turns a near-zero gradient's sign flip into a step of up to 2 lr
    err = np.abs(gb - ga)
    assert np.mean(err <= 1e-6 + 1e-5 * np.abs(ga)) >= 0.97
    assert err.max() <= 2 * 5e-2 * len(seq)


def test_train_steps_host_u8_matches_dequantized_float_images():
    """8-bit host images (the PPM bytes the reference loads, image.cpp:60-79)
    train exactly like their FP32 dequantization (byte / 255, image.cpp:21-27)."""
    s, init = toy_scene(seed=6)
    seq = orc.view_sequence(1, 0, len(s.views), 7)
    ims = s.images()
    q = [np.round(np.clip(ims[v], 0.0, 1.0) * 255.0).astype(np.uint8) for v in seq]  # quantize, image.cpp:12-19
    cams = [dev_cam(s.views[v]) for v in seq]
    a = device_trainer(init, s)
    la = a.train_steps_host(cams, [(b.astype(np.float64) / 255.0).astype(np.float32) for b in q])
    b8 = device_trainer(init, s)
    lb = b8.train_steps_host_u8(cams, q)
    np.testing.assert_allclose(lb, la, rtol=1e-6)
    ca, cb = a.download_cloud(), b8.download_cloud()
    ga = np.concatenate([ca["pos"], ca["rot"], ca["ls"], ca["feat"], ca["op"][:, None]], 1)
    gb = np.concatenate([cb["pos"], cb["rot"], cb["ls"], cb["feat"], cb["op"][:, None]], 1)
    err = np.abs(gb - ga)
    assert np.mean(err <= 1e-6 + 1e-5 * np.abs(ga)) >= 0.97
