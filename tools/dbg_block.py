"""Per-step stage times and counters of chosen blocks of a K-block cfg 3 plan
(diagnostics for tools/blocks_bench.py outliers).

usage: python tools/dbg_block.py --blocks-k 8 --which 1,0 [--steps 40]
"""
import argparse
import sys

import numpy as np

sys.path.insert(0, '/root/repo')
from paper_2405_13943_b200 import api  # noqa: E402
from paper_2405_13943_b200.scene import aerial_scene, perturbed_init  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--blocks-k", type=int, default=8)
ap.add_argument("--which", default="1,0")
ap.add_argument("--steps", type=int, default=40)
args = ap.parse_args()
cfg = dict(n=6_000_000, width=1600, height=1066, views=96, scale=1.4)
cloud, cams = aerial_scene(cfg["n"], cfg["width"], cfg["height"], cfg["views"], 100.0, 42)
init = perturbed_init(cloud, 42)
centers = np.array([c.center() for c in cams])
plan = api.Plan(cloud["ids"], cloud["pos"], centers, args.blocks_k, cfg["scale"])
for b in [int(x) for x in args.which.split(",")]:
    ids, views = plan.block(b)
    sel = ids.astype(np.int64)
    blk = api.Block(0, 3)
    blk.upload_cloud(init["ids"][sel], init["pos"][sel], init["rot"][sel], init["ls"][sel], init["feat"][sel], init["op"][sel])
    vcams = [cams[v].device() for v in views]
    blk.set_views(vcams, [np.full((cfg["height"], cfg["width"], 3), 0.5) for _ in vcams])
    blk.trainer_init(api.trainer_config(iterations=30000, densify={"enabled": 0}))
    blk.enable_stage_timing(True)
    g = np.random.default_rng(7)
    seq = [int(v) for v in g.integers(0, len(vcams), args.steps)]
    for s, vi in enumerate(seq):
        blk.train_steps([vi], want_losses=False)
        st = blk.stage_times()
        c = blk.step_counters()
        big = {k: round(v, 3) for k, v in st.items() if v > 0.05}
        print(b, s, vi, views[vi], c['visible'], c['pairs'], c['launches'], round(sum(st.values()), 3), big, flush=True)
    blk.close()
