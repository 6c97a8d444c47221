"""A run of every device entry point for the checked library
(lib/libbsgpu_checked.so: device invariant checks on, tests/test_gpu_checked.py):
projection (global path), render (per-tile path and the crowded-tile
switch), render backward, the loss kernels on given images, train steps with
densification across a pending asynchronous round, evaluation, the GSPL
encode, the owner table, and two training steps of the cfg 2 bench block at
full size. Test infrastructure only."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
sys.path.insert(0, HERE)

from paper_2405_13943_b200 import api  # noqa: E402
from paper_2405_13943_b200.scene import aerial_scene  # noqa: E402


def main():
    cloud, cams = aerial_scene(3000, 96, 64, 4, 20.0, 3, tilt_deg=30.0)
    dc = [c.device() for c in cams]
    b = api.Block(0, 3)
    b.upload_cloud(cloud["ids"], cloud["pos"], cloud["rot"], cloud["ls"], cloud["feat"], cloud["op"])
    b.project(dc[0])
    b.tile_pairs()
    gts = [b.render(c)[0] for c in dc]
    g = np.random.default_rng(1)
    b.render_backward(dc[1], np.clip(gts[1] + 0.1 * g.standard_normal(gts[1].shape), 0, 1))
    b.image_loss(gts[0], gts[1])
    b.set_views(dc, gts)
    b.trainer_init(api.trainer_config(iterations=40, densify=dict(enabled=1, interval=3, stop_iteration=6,
                                                                  grad_threshold=1e-9, prune_opacity=0.3)))
    rows = list(range(0, b.n, 7))
    b.set_shared(rows, list(range(len(rows))), [1] * len(rows), [1] * len(rows))
    x = b.download_cloud()
    z = np.concatenate([x["pos"], x["rot"], x["ls"], x["feat"], x["op"][:, None]], 1)[rows]
    b.set_anchor(z, z, api.penalties())
    b.train_steps([0, 1, 2])
    b.consensus_round_async(1.6, True, iteration=3, diagnostics=True)
    b.train_steps([3, 0, 1, 2])  # crosses the densification at iteration 6 with the round pending
    b.consensus_wait()
    b.evaluate(dc, gts, 2)
    b.encode_gspl()
    # a crowded tile: more than 2048 pairs take the global sorts
    n = 3000
    pos = np.column_stack([g.uniform(-0.4, 0.4, n), g.uniform(-0.4, 0.4, n), g.uniform(4.0, 6.0, n)])
    q = g.normal(size=(n, 4))
    c = api.Block(0, 3)
    c.upload_cloud(np.arange(n, dtype=np.uint64), pos, q / np.linalg.norm(q, axis=1, keepdims=True),
                   np.full((n, 3), -4.0), g.uniform(0, 1, (n, 3)), g.normal(size=n) - 3.0)
    cam = api.make_camera(50, 50, 8, 8, np.eye(3), np.zeros(3), 16, 16)
    c.render(cam)
    c.render(cam)
    # the owner table
    t = api.OwnerTable([3, 5, 9], [3, 6, 5], 3)
    t.remove([[3], [5, 7], [9]])
    t.close()
    # the bench block at full size (2M rows, 1024x768): per-tile binning at scale
    cloud, cams = aerial_scene(2_000_000, 1024, 768, 4, 100.0, 42)
    dc = [cc.device() for cc in cams]
    d = api.Block(0, 3)
    d.upload_cloud(cloud["ids"], cloud["pos"], cloud["rot"], cloud["ls"], cloud["feat"], cloud["op"])
    gts = [d.render(cc)[0] for cc in dc]
    d.set_views(dc, gts)
    d.trainer_init(api.trainer_config(iterations=100, densify={"enabled": 0}))
    d.train_steps([0, 1, 2, 3])
    d.synchronize()
    print("checked workload done")


if __name__ == "__main__":
    main()
