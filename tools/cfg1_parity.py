"""BASELINE.json configs[0] end to end: the reference generator verbatim
(generate_scene seed 42, 200k GT Gaussians, 32 views at 256x256), the
reference's init_cloud_from_points (100k points), plan_cluster(K=2, s=1.4,
holdout 8), 100 iterations, consensus every 10, alpha 1.6 (and alpha 1 for the
dual-mean check). Runs the oracle's run_simulated (FP64 CPU, test
infrastructure) and the device run_simulated on the same inputs, and compares
holdout PSNR (both models evaluated by the same FP64 renderer), per-round
diagnostics and wall time. Writes one JSON document.

usage: python tools/cfg1_parity.py [--out profiles/cfg1_parity.json] [--alphas 1.6,1.0] [--gaussians 200000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import _oracle as orc  # noqa: E402
from paper_2405_13943_b200 import api  # noqa: E402
from refcases import HostCloud  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "cfg1_parity.json"))
    ap.add_argument("--alphas", default="1.6,1.0")
    ap.add_argument("--gaussians", type=int, default=200000)
    ap.add_argument("--iterations", type=int, default=100)
    ap.add_argument("--interval", type=int, default=10)
    args = ap.parse_args()
    t0 = time.time()
    sc = orc.SynthConfig()
    sc.seed, sc.gaussians, sc.cameras, sc.image_size, sc.extent = 42, args.gaussians, 32, 256, 10.0
    scene = orc.generate_scene(sc)
    t_gen = time.time() - t0
    p, c = scene.points()
    t1 = time.time()
    init = HostCloud.from_oracle(orc.init_cloud_from_points(p, c, 0, 0.1)).narrowed()
    t_init = time.time() - t1
    scene.has_checkpoint = True
    scene.checkpoint = init.oracle()
    images = scene.images()
    views = scene.views
    cams = [api.make_camera(v.fx, v.fy, v.cx, v.cy, v.R, v.t, v.width, v.height) for v in views]

    def holdout_psnr(model):
        vals = [orc.psnr(orc.render(model, v, orc.RenderConfig())[0], images[i])
                for i, v in enumerate(views) if i % 8 == 0]
        return float(np.mean(vals)), [float(x) for x in vals]

    out = {"config": {"generator": "generate_scene(seed=42, gaussians=%d, cameras=32, image_size=256, extent=10)"
                      % args.gaussians, "init_points": int(init.n), "blocks": 2, "expand_scale": 1.4,
                      "holdout": 8, "iterations": args.iterations, "interval": args.interval, "trainer_seed": 7},
           "setup_seconds": {"generate_scene": t_gen, "init_cloud_from_points": t_init}, "runs": []}
    for alpha in [float(a) for a in args.alphas.split(",")]:
        tc = orc.TrainerConfig()
        tc.iterations, tc.seed = args.iterations, 7
        tc.densify_enabled = False  # inert at 100 iterations (interval 200), trainer.cpp:301-304
        plan = orc.plan_cluster(scene, 2, 1.4, 8, tc)
        so = orc.SessionOptions()
        so.total_iterations = args.iterations
        so.consensus.interval = args.interval
        so.consensus.alpha = alpha
        t2 = time.time()
        want = orc.run_simulated(plan, tc, so)
        cpu_wall = time.time() - t2
        sess = api.session_options(args.iterations, interval=args.interval, alpha=alpha, blocks=2, expand_scale=1.4,
                                   holdout=8, seed=7)
        cloud = dict(ids=init.ids, pos=init.pos, rot=init.rot, ls=init.ls, feat=init.feat, op=init.op)
        t3 = time.time()
        model, rounds, gpu_wall = api.run_simulated(cloud, cams, images, api.trainer_config(iterations=args.iterations),
                                                    sess)
        gpu_call = time.time() - t3
        mc = HostCloud(model["ids"], model["pos"], model["rot"], model["ls"], model["feat"], model["op"])
        p_gpu, pv_gpu = holdout_psnr(mc.oracle())
        p_cpu, pv_cpu = holdout_psnr(want.model)
        p_init, _ = holdout_psnr(init.oracle())
        rd = []
        for g, w in zip(rounds, want.rounds):
            rd.append({"iteration": g["iteration"], "gpu": {k: g[k] for k in ("primal", "dual", "max_disagreement",
                                                                              "dual_mean_linf", "mean_loss")},
                       "cpu": {"primal": w.primal_residual, "dual": w.dual_residual,
                               "max_disagreement": w.max_disagreement, "dual_mean_linf": w.dual_mean_linf,
                               "mean_loss": w.mean_loss},
                       "rho_p_equal": g["rho"][0] == w.rho.rho_p})
        run = {"alpha": alpha, "psnr_gpu": p_gpu, "psnr_cpu_ref": p_cpu, "psnr_delta_db": p_gpu - p_cpu,
               "psnr_init": p_init, "psnr_per_view_gpu": pv_gpu, "psnr_per_view_cpu": pv_cpu,
               "cpu_wall_seconds": cpu_wall, "cpu_iters_per_sec": args.iterations / cpu_wall,
               "gpu_wall_seconds": gpu_wall, "gpu_call_seconds": gpu_call,
               "gpu_iters_per_sec": args.iterations / gpu_wall, "shared_ids": rounds[-1]["shared_count"],
               "rounds": rd}
        out["runs"].append(run)
        print(json.dumps({k: v for k, v in run.items() if k != "rounds"}), flush=True)
    out["host"] = {"nproc": os.cpu_count()}
    try:
        out["host"]["cpu_model"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if "model name" in l][0]
    except Exception:
        pass
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
