"""BASELINE configs[0] end to end as a test (SURVEY §8(d) cfg 1): the
reference generator verbatim (generate_scene seed 42, 200k ground-truth
Gaussians, 32 views at 256x256, synth.cpp:13-77), the reference's
init_cloud_from_points (100k points), plan_cluster(K=2, s=1.4, holdout 8),
100 iterations with consensus every 10 (runtime.cpp:256-263,482-671), at
alpha = 1.6 and alpha = 1. The oracle's FP64 run_simulated and the device's
run_simulated get identical inputs; both final models are scored by the same
FP64 renderer on the holdout views (metrics.cpp:14-51).

Bars: holdout PSNR within 0.1 dB; the same penalty adaptation
decision in every round (rho_p equal, admm.cpp:200-217); the dual mean at
alpha = 1 vanishes (acceptance crit. 4; FP32 analogue 1e-5 of the reference's
1e-9); residuals per round within 1e-2 relative (they are sums of FP32 vs FP64
rows after 10 Adam steps)."""
import threading

import numpy as np
import pytest

import _oracle as orc
from gpu_helpers import gpu
from paper_2405_13943_b200 import api
from refcases import HostCloud

pytestmark = gpu

ITERS, INTERVAL = 100, 10


@pytest.fixture(scope="module")
def cfg1():
    sc = orc.SynthConfig()
    sc.seed, sc.gaussians, sc.cameras, sc.image_size, sc.extent = 42, 200000, 32, 256, 10.0
    scene = orc.generate_scene(sc)
    p, c = scene.points()
    init = HostCloud.from_oracle(orc.init_cloud_from_points(p, c, 0, 0.1)).narrowed()
    scene.has_checkpoint = True
    scene.checkpoint = init.oracle()
    # both alphas' oracle runs (FP64, K worker threads each, GIL released) in parallel
    runs = {}

    def oracle_run(alpha):
        tc = orc.TrainerConfig()
        tc.iterations, tc.seed = ITERS, 7
        tc.densify_enabled = False  # inert at 100 iterations (interval 200), trainer.cpp:301-304
        plan = orc.plan_cluster(scene, 2, 1.4, 8, tc)
        so = orc.SessionOptions()
        so.total_iterations = ITERS
        so.consensus.interval = INTERVAL
        so.consensus.alpha = alpha
        runs[alpha] = orc.run_simulated(plan, tc, so)

    threads = [threading.Thread(target=oracle_run, args=(a,)) for a in (1.6, 1.0)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    return scene, init, runs


def holdout_psnr(model, views, images):
    return float(np.mean([orc.psnr(orc.render(model, v, orc.RenderConfig())[0], images[i])
                          for i, v in enumerate(views) if i % 8 == 0]))


@pytest.mark.parametrize("alpha", [1.6, 1.0])
def test_cfg1_run_matches_cpu_reference(cfg1, alpha):
    scene, init, runs = cfg1
    want = runs[alpha]
    images, views = scene.images(), scene.views
    cams = [api.make_camera(v.fx, v.fy, v.cx, v.cy, v.R, v.t, v.width, v.height) for v in views]
    sess = api.session_options(ITERS, interval=INTERVAL, alpha=alpha, blocks=2, expand_scale=1.4, holdout=8, seed=7)
    cloud = dict(ids=init.ids, pos=init.pos, rot=init.rot, ls=init.ls, feat=init.feat, op=init.op)
    model, rounds, _ = api.run_simulated(cloud, cams, images, api.trainer_config(iterations=ITERS), sess)
    mc = HostCloud(model["ids"], model["pos"], model["rot"], model["ls"], model["feat"], model["op"])
    p_gpu = holdout_psnr(mc.oracle(), views, images)
    p_cpu = holdout_psnr(want.model, views, images)
    p_init = holdout_psnr(init.oracle(), views, images)
    assert p_cpu > p_init + 1.0  # the run trains
    assert abs(p_gpu - p_cpu) <= 0.1, (p_gpu, p_cpu)
    assert np.array_equal(model["ids"], want.model.dict()["ids"])
    assert len(rounds) == len(want.rounds) == ITERS // INTERVAL
    for g, w in zip(rounds, want.rounds):
        assert g["iteration"] == w.iteration
        assert g["rho"][0] == w.rho.rho_p  # same adaptation decisions
        assert g["primal"] == pytest.approx(w.primal_residual, rel=1e-2)
        assert g["dual"] == pytest.approx(w.dual_residual, rel=1e-2, abs=1e-9)
        assert g["mean_loss"] == pytest.approx(w.mean_loss, rel=1e-2)
        if alpha == 1.0:
            assert g["dual_mean_linf"] <= 1e-5
