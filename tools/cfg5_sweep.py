"""BASELINE.json configs[4] (SURVEY §8(d) cfg 5): single-block (K = 1) training
throughput sweep, N in {1, 2, 4, 8, 16}M Gaussians, one 1920x1080 view that
sees nearly the whole scene, constant-0.5 ground truth (throughput only).
20 warm-up + 100 timed iterations (CUDA events on the block's stream, no
per-stage events), then a 50-iteration pass with per-stage CUDA events.

usage: python tools/cfg5_sweep.py [--sizes 1,2,4,8,16] [--out profiles/cfg5_sweep.json]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2405_13943_b200 import api  # noqa: E402
from paper_2405_13943_b200.scene import aerial_scene, look_at  # noqa: E402

W, H, EXTENT = 1920, 1080, 100.0


def overview_camera():
    """Altitude 150 m over the scene centre, 5 degrees off nadir, f = 0.8 W:
    the 100 m x 100 m slab fills the 1920x1080 frame."""
    alt, tilt = 150.0, 5.0
    d = alt * math.tan(math.radians(tilt))
    f = 0.8 * W
    return look_at([0.0, alt, 0.0], [d, 0.0, 0.0], [0.0, 1.0, 0.0], f, f, W / 2, H / 2, W, H)


def run(n, warmup, steps, stage_steps):
    import torch

    cloud, _ = aerial_scene(n, W, H, 1, EXTENT, 42)
    cam = overview_camera().device()
    blk = api.Block(0, 3)
    blk.upload_cloud(cloud["ids"], cloud["pos"], cloud["rot"], cloud["ls"], cloud["feat"], cloud["op"])
    del cloud
    blk.set_views([cam], [np.full((H, W, 3), 0.5)])
    blk.trainer_init(api.trainer_config(iterations=30000, densify={"enabled": 0}))
    stream = torch.cuda.ExternalStream(blk.stream())
    for _ in range(warmup):
        blk.train_steps([0], want_losses=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = blk.launch_count()
    e0.record(stream)
    for _ in range(steps):
        blk.train_steps([0], want_losses=False)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    launches = (blk.launch_count() - l0) / steps
    blk.enable_stage_timing(True)
    acc, vis, pairs = {}, 0, 0
    for _ in range(stage_steps):
        blk.train_steps([0], want_losses=False)
        for k, v in blk.stage_times().items():
            acc[k] = acc.get(k, 0.0) + v
        c = blk.step_counters()
        vis += c["visible"]
        pairs += c["pairs"]
    blk.close()
    return {"gaussians": n, "width": W, "height": H, "ms_per_iter": ms, "iters_per_s": 1000.0 / ms,
            "launches_per_iter": launches, "visible": vis / stage_steps, "pairs": pairs / stage_steps,
            "stage_ms": {k: round(v / stage_steps, 4) for k, v in acc.items()}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1,2,4,8,16")
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--stage-steps", type=int, default=50)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "cfg5_sweep.json"))
    args = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    rows = []
    for s in args.sizes.split(","):
        n = int(float(s) * 1_000_000)
        t0 = time.time()
        r = run(n, args.warmup, args.steps, args.stage_steps)
        r["wall_s"] = round(time.time() - t0, 1)
        print(json.dumps(r), flush=True)
        rows.append(r)
    doc = {"config": "BASELINE configs[4]: K=1 block, one 1920x1080 overview view, constant-0.5 GT, SH degree 0, "
                     "densification off; N Gaussians from the cfg2 generator (100 m box)",
           "gpu": torch.cuda.get_device_name(0), "rows": rows}
    with open(args.out, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
