import sys, json, numpy as np
sys.path.insert(0, '/root/repo')
import torch
from paper_2405_13943_b200 import api
from paper_2405_13943_b200.scene import aerial_scene, perturbed_init
cfg = dict(n=6_000_000, width=1600, height=1066, views=96, scale=1.4)
cloud, cams = aerial_scene(cfg["n"], cfg["width"], cfg["height"], cfg["views"], 100.0, 42)
init = perturbed_init(cloud, 42)
centers = np.array([c.center() for c in cams])
plan = api.Plan(cloud["ids"], cloud["pos"], centers, 8, cfg["scale"])
for b in (5, 6, 0):
    ids, views = plan.block(b)
    sel = ids.astype(np.int64)
    blk = api.Block(0, 3)
    blk.upload_cloud(init["ids"][sel], init["pos"][sel], init["rot"][sel], init["ls"][sel], init["feat"][sel], init["op"][sel])
    vcams = [cams[v].device() for v in views]
    blk.set_views(vcams, [np.full((cfg["height"], cfg["width"], 3), 0.5) for _ in vcams])
    blk.trainer_init(api.trainer_config(iterations=30000, densify={"enabled": 0}))
    blk.enable_stage_timing(True)
    for vi in range(len(vcams)):
        blk.train_steps([vi], want_losses=False)
        st = blk.stage_times(); c = blk.step_counters()
        big = {k: round(v, 3) for k, v in st.items() if v > 0.3}
        print(b, vi, views[vi], c['visible'], c['pairs'], c['launches'], round(sum(st.values()), 3), big, flush=True)
    blk.close()
