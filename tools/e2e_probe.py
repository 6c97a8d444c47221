"""e2e diagnostic: bsg_train_steps_host_u8 throughput against the number of
steps per call (the bench's e2e leg uses one call per consensus interval)."""
import time

import numpy as np
import torch

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

torch.cuda.set_device(0)
cfg = bench.CFGS["cfg3"]
blk, cams, gts, _ = bench.build_block(cfg, 0, 1, 0)
pinned = [torch.from_numpy(np.clip(np.rint(np.clip(x, 0.0, 1.0) * 255.0), 0, 255).astype(np.uint8)).pin_memory()
          for x in gts]
stream = torch.cuda.ExternalStream(blk.stream())
g = np.random.default_rng(5)
seq = [int(v) for v in g.integers(0, len(cams), 400)]
for v in seq[:10]:
    blk.train_steps([v], want_losses=False)
torch.cuda.synchronize()


def dev(n):
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for v in seq[:n]:
        blk.train_steps([v], want_losses=False)
    f1.record(stream)
    torch.cuda.synchronize()
    return f0.elapsed_time(f1) / n


def e2e(n, chunk):
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    f0.record(stream)
    for i in range(0, n, chunk):
        vs = seq[i:i + chunk]
        blk.train_steps_host_u8([cams[v] for v in vs], [pinned[v].numpy() for v in vs])
    f1.record(stream)
    torch.cuda.synchronize()
    return f0.elapsed_time(f1) / n, (time.perf_counter() - t0) * 1e3 / n


print("device ms/step", round(dev(200), 4))
for chunk in (1, 5, 25, 100, 200):
    print("e2e chunk", chunk, [round(x, 4) for x in e2e(200, chunk)])
print("device ms/step", round(dev(200), 4))
