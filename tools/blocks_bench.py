"""Per-block step times of a K-block plan, measured one block at a time on one
GPU (blocks map one-to-one to GPUs).

For BASELINE configs[1]-[3] shapes: plan the scene into K blocks with the
native planner, then for every block b build its device context (its rows,
its training views, constant-0.5 ground truth: throughput only), warm up and
time `--steps` training steps with CUDA events. On K GPUs the blocks step
concurrently, so the K-GPU iteration time is bounded below by the slowest
block; `projected_iters_per_s` = 1000 / max_b(ms_b) is that bound, NOT a
multi-GPU measurement (this run has one GPU; consensus is measured separately
by tools/consensus_bench.py). Densification off.

usage: python tools/blocks_bench.py --config cfg2 --blocks 2,4,8 [--out profiles/blocks_cfg2.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2405_13943_b200 import api  # noqa: E402
from paper_2405_13943_b200.scene import aerial_scene, perturbed_init  # noqa: E402

CONFIGS = {
    "cfg2": dict(n=2_000_000, width=1024, height=768, views=64, scale=1.4),
    "cfg3": dict(n=6_000_000, width=1600, height=1066, views=96, scale=1.4),
    "cfg4": dict(n=20_000_000, width=1600, height=1066, views=96, scale=2.0),
}


def time_block(init, sel, cams, views, cfg, steps, warmup):
    import torch
    blk = api.Block(0, 3)
    blk.upload_cloud(init["ids"][sel], init["pos"][sel], init["rot"][sel], init["ls"][sel], init["feat"][sel],
                     init["op"][sel])
    vcams = [cams[v].device() for v in views]
    blk.set_views(vcams, [np.full((cfg["height"], cfg["width"], 3), 0.5) for _ in vcams])
    blk.trainer_init(api.trainer_config(iterations=30000, densify={"enabled": 0}))
    g = np.random.default_rng(7)
    seq = [int(v) for v in g.integers(0, len(vcams), warmup + steps)]
    for v in seq[:warmup]:
        blk.train_steps([v], want_losses=False)
    stream = torch.cuda.ExternalStream(blk.stream())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for v in seq[warmup:]:
        blk.train_steps([v], want_losses=False)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    blk.close()
    return ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--blocks", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    cfg = CONFIGS[args.config]
    cloud, cams = aerial_scene(cfg["n"], cfg["width"], cfg["height"], cfg["views"], 100.0, 42)
    init = perturbed_init(cloud, 42)
    centers = np.array([c.center() for c in cams])
    rows = []
    for k in [int(x) for x in args.blocks.split(",")]:
        t0 = time.time()
        plan = api.Plan(cloud["ids"], cloud["pos"], centers, k, cfg["scale"])
        sids, _, _ = plan.shared()
        per = []
        for b in range(k):
            ids, views = plan.block(b)
            ms = time_block(init, ids.astype(np.int64), cams, views, cfg, args.steps, args.warmup)
            per.append(dict(block=b, gaussians=int(len(ids)), views=int(len(views)), ms_per_step=ms))
        mx = max(p["ms_per_step"] for p in per)
        row = dict(blocks=k, shared_slots=int(len(sids)), per_block=per, max_ms=mx,
                   mean_ms=float(np.mean([p["ms_per_step"] for p in per])),
                   projected_iters_per_s=1000.0 / mx, wall_s=round(time.time() - t0, 1))
        print(json.dumps(row), flush=True)
        rows.append(row)
    doc = {"config": args.config, **cfg, "note": "per-block steps timed one block at a time on one GPU; "
           "projected_iters_per_s = 1000 / slowest block (a bound for K GPUs, not a multi-GPU measurement)",
           "gpu": torch.cuda.get_device_name(0), "rows": rows}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
