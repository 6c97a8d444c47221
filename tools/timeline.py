"""Kernel timeline of the bench workload (cfg 3 headline, one block) from CUPTI via
torch.profiler: per-kernel warm durations, GPU idle gaps between consecutive
kernels of one step, and the busy fraction of the step. Answers "how much of
the step is launch / host-sync gap rather than kernel time".

usage: python tools/timeline.py [--steps 50] [--out profiles/timeline.json]
"""
import argparse
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--out", default=None)
    ap.add_argument("--e2e", action="store_true", help="steps through bsg_train_steps_host_u8 (pinned 8-bit host GT)")
    ap.add_argument("--config", default="cfg3")
    args = ap.parse_args()
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    torch.cuda.set_device(0)
    cfg = bench.CFGS[args.config]
    blk, cams, gts, _ = bench.build_block(cfg, 0, 1, 0)
    g = np.random.default_rng(3)
    seq = [int(v) for v in g.integers(0, len(cams), args.warmup + args.steps)]
    if args.e2e:
        pinned = [torch.from_numpy(np.clip(np.rint(np.clip(x, 0.0, 1.0) * 255.0), 0, 255).astype(np.uint8)).pin_memory()
                  for x in gts]

        def step(v):
            blk.train_steps_host_u8([cams[v]], [pinned[v].numpy()])

        def chunk(vs):  # the bench's e2e path: one host-image call per consensus interval
            blk.train_steps_host_u8([cams[v] for v in vs], [pinned[v].numpy() for v in vs])
    else:
        def step(v):
            blk.train_steps([v], want_losses=False)
    for v in seq[:args.warmup]:
        step(v)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        if args.e2e:
            rest = seq[args.warmup:]
            for i in range(0, len(rest), 25):
                chunk(rest[i:i + 25])
        else:
            for v in seq[args.warmup:]:
                step(v)
        torch.cuda.synchronize()
    # host launch -> device start latency per kernel (chrome trace: correlation ids)
    import tempfile
    with tempfile.NamedTemporaryFile(suffix=".json", delete=False) as tf:
        trace_path = tf.name
    prof.export_chrome_trace(trace_path)
    with open(trace_path) as f:
        tr = json.load(f)
    os.unlink(trace_path)
    launches, kernels = {}, {}
    for e in tr.get("traceEvents", []):
        cat = e.get("cat", "")
        corr = (e.get("args") or {}).get("correlation")
        if corr is None or e.get("ph") != "X":
            continue
        if cat == "cuda_runtime" or cat == "cuda_driver":
            launches[corr] = (e["ts"], e["ts"] + e.get("dur", 0), e.get("name", ""))
        elif cat in ("kernel", "gpu_memset", "gpu_memcpy"):
            kernels[corr] = (e["ts"], e["ts"] + e.get("dur", 0), e.get("name", ""))
    slack = defaultdict(list)
    rows = sorted((ks, kn, ks - launches[corr][1]) for corr, (ks, ke, kn) in kernels.items() if corr in launches)
    pos = 0
    for ks, kn, sl in rows:
        short = kn.replace("bsg::(anonymous namespace)::", "").replace("void ", "").split("(")[0]
        if short.startswith("zero_counters"):
            pos = 0
        slack[f"{pos:02d} {short}"].append(sl)  # > 0: the kernel was queued before it could start
        pos += 1
    host_slack = {k: {"median_us": float(np.median(v)), "min_us": float(np.min(v)), "n": len(v)}
                  for k, v in slack.items()}
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    kern = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev], key=lambda t: t[0])
    if not kern:
        print(json.dumps({"error": "no CUDA activity captured"}))
        return
    t0, t1 = kern[0][0], kern[-1][1]
    span = t1 - t0
    busy = 0.0
    gaps = []
    cur_end = kern[0][0]
    per = defaultdict(lambda: [0, 0.0])
    prev_name = None
    for s, e, n in kern:
        if s > cur_end:
            gaps.append((s - cur_end, prev_name, n))
        busy += max(0.0, e - max(s, cur_end))
        cur_end = max(cur_end, e)
        per[n][0] += 1
        per[n][1] += e - s
        prev_name = n
    gap_by = defaultdict(lambda: [0, 0.0])
    for d, a, b in gaps:
        k = f"{a[:40]} -> {b[:40]}"
        gap_by[k][0] += 1
        gap_by[k][1] += d
    top_gaps = sorted(gap_by.items(), key=lambda kv: -kv[1][1])[:12]
    # one step in order (from the 10th preprocess launch to the next)
    starts = [i for i, k in enumerate(kern) if "preprocess_kernel" in k[2]]
    seq_one = []
    if len(starts) > 11:
        prev_end = kern[starts[10] - 1][1]
        for s, e, n in kern[starts[10]:starts[11]]:
            short = n.replace("bsg::(anonymous namespace)::", "").replace("void ", "").split("(")[0]
            seq_one.append({"kernel": short, "gap_us": round(s - prev_end, 2), "us": round(e - s, 2)})
            prev_end = e
    out = {
        "steps": args.steps,
        "one_step": seq_one,
        "launch_to_start_us": host_slack,
        "span_us_per_step": span / args.steps,
        "busy_us_per_step": busy / args.steps,
        "idle_us_per_step": (span - busy) / args.steps,
        "kernels_per_step": len(kern) / args.steps,
        "kernels": {n: {"per_step": c / args.steps, "us_per_step": t / args.steps}
                    for n, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1])},
        "top_gaps": [{"between": k, "per_step": c / args.steps, "us_per_step": t / args.steps}
                     for k, (c, t) in top_gaps],
        "gpu": torch.cuda.get_device_name(0),
    }
    print(json.dumps(out, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
    blk.close()


if __name__ == "__main__":
    main()
