"""Consensus cost on one GPU (SURVEY §8(d) "ADMM consensus ms/iter", §8(e)).

Builds BASELINE configs[2] (6M Gaussians, 1600x1066, K=8, s=1.4) or
configs[3] (20M, K=8, s=2.0) with the cfg2 generator, plans the K blocks on
the host (bit-exact planner) and runs block 0 alone on this GPU with its real
shared set and global slot table. With one rank the NCCL AllReduce is skipped,
so what is timed is every device kernel of the round (slot owner counts are
set to 1 so the single rank's z stays its own relaxed parameters and the
training cost is unperturbed; sign pre-pass, relaxed
pack, unpack / dual update / residuals, penalty adaptation) plus the overlap
with the next step; the AllReduce payload is reported in bytes, with its time
at NVLink 5 nominal bandwidth given as an estimate only (not measured: this
run has one GPU). Ground truth is a constant image (throughput only).

usage: python tools/consensus_bench.py [--config cfg3|cfg4] [--interval 25] [--out profiles/consensus_cfg3.json]
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
    "cfg3": dict(n=6_000_000, width=1600, height=1066, views=96, k=8, scale=1.4),
    "cfg4": dict(n=20_000_000, width=1600, height=1066, views=96, k=8, scale=2.0),
}
NVLINK5_GBS = 900.0  # per direction, nominal


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--interval", type=int, default=25)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--out", default=None)
    ap.add_argument("--profile", action="store_true",
                    help="also: per-kernel GPU time per step with and without asynchronous rounds (CUPTI)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    import torch
    torch.cuda.set_device(0)
    t0 = time.time()
    cloud, cams = aerial_scene(cfg["n"], cfg["width"], cfg["height"], cfg["views"], 100.0, 42)
    init = perturbed_init(cloud, 42)
    centers = np.array([c.center() for c in cams])
    plan = api.Plan(cloud["ids"], cloud["pos"], centers, cfg["k"], cfg["scale"])
    ids, views = plan.block(0)
    sids, cnt, _ = plan.shared()
    rows, slots, first = plan.block_shared(0)
    sel = ids.astype(np.int64)
    t_plan = time.time() - t0
    blk = api.Block(0, 3)
    blk.upload_cloud(init["ids"][sel], init["pos"][sel], init["rot"][sel], init["ls"][sel], init["feat"][sel],
                     init["op"][sel])
    vcams = [cams[v].device() for v in views]
    blk.set_views(vcams, [np.full((cfg["height"], cfg["width"], 3), 0.5) for _ in vcams])
    blk.trainer_init(api.trainer_config(iterations=30000, densify={"enabled": 0}))
    # one rank holds only its own contributions: with the plan's owner counts
    # z = (own contribution) / owners would drag the anchors away and change the
    # training cost, so every slot counts one owner here (same kernels, same sizes)
    blk.set_shared(rows, slots, np.ones_like(first), np.ones_like(cnt))
    init_rows = np.concatenate([init["pos"], init["rot"], init["ls"], init["feat"], init["op"][:, None]], 1)
    zprev = init_rows[sids.astype(np.int64)]
    blk.set_anchor(zprev[slots], zprev, api.penalties())
    del cloud, init, init_rows
    nv = len(vcams)
    stream = torch.cuda.ExternalStream(blk.stream())
    g = np.random.default_rng(1)
    seq = [int(v) for v in g.integers(0, nv, 40 + 4 * args.steps)]
    pos = [0]

    def step():
        blk.train_steps([seq[pos[0]]], want_losses=False)
        pos[0] += 1

    def timed(fn, n):
        pos[0] = 40  # every variant replays the same view sequence
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn(n)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for _ in range(10):
        step()
    # warm-up rounds (first launches of the round's kernels, lazy module loading)
    for _ in range(2):
        blk.consensus_round_async(1.6, True, iteration=0)
        step()
        blk.consensus_wait()
        blk.consensus_round(1.6, True)
        step()
    # Windows of `interval` steps in rotation: no round / an asynchronous
    # round at the start (waited after the window's first step) / a
    # synchronous round at the start. The model keeps training, so the
    # rotation keeps every variant on the same state (timing the variants one
    # after the other measured the drift of the step cost as consensus cost).
    rounds_async, rounds_sync = [], []
    tot = {"plain": 0.0, "async": 0.0, "sync": 0.0}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    windows = max(1, args.steps // args.interval)
    pos[0] = 40
    for w in range(3 * windows):
        kind = ("plain", "async", "sync")[w % 3]
        if kind == "plain":
            start = pos[0] if pos[0] + args.interval <= len(seq) else 40
        pos[0] = start  # the three windows of a rotation render the same views
        torch.cuda.synchronize()
        e0.record(stream)
        if kind == "async":
            blk.consensus_round_async(1.6, True, iteration=w)
        elif kind == "sync":
            rounds_sync.append(blk.consensus_round(1.6, True))
        for j in range(args.interval):
            step()
            if kind == "async" and j == 0:
                rounds_async.append(blk.consensus_wait())
        e1.record(stream)
        torch.cuda.synchronize()
        tot[kind] += e0.elapsed_time(e1)
    n_w = windows * args.interval
    ms_plain, ms_async, ms_sync = tot["plain"] / n_w, tot["async"] / n_w, tot["sync"] / n_w

    def with_async(n):  # (for --profile)
        pending = False
        for i in range(1, n + 1):
            step()
            if pending:
                blk.consensus_wait()
                pending = False
            if i % args.interval == 0:
                blk.consensus_round_async(1.6, True, iteration=i)
                pending = True
        if pending:
            blk.consensus_wait()

    D = 14
    S = len(sids)
    payload = 4 * 4 * S + 4 * (D + 1) * S + 8 * 3  # q pre-pass + relaxed contributions/flags + residual scalars
    K = cfg["k"]
    est_ms = 2 * (K - 1) / K * payload / (NVLINK5_GBS * 1e9) * 1e3
    round_ms = float(np.mean([r["ms"] for r in rounds_async])) if rounds_async else None
    out = {
        "config": args.config, **cfg, "interval": args.interval, "steps": args.steps,
        "block0_gaussians": int(len(ids)), "block0_views": int(nv), "block0_shared_rows": int(len(rows)),
        "global_shared_slots": int(S), "shared_fraction_of_n": S / cfg["n"],
        "ms_per_step_no_consensus": ms_plain,
        "ms_per_step_async_rounds": ms_async,
        "ms_per_step_sync_rounds": ms_sync,
        "round_device_ms_kernels_only": round_ms,
        "consensus_ms_per_iter_exposed_async": ms_async - ms_plain,
        "consensus_ms_per_iter_exposed_sync": ms_sync - ms_plain,
        "allreduce_payload_bytes_per_round": payload,
        "allreduce_ms_estimate_nvlink5_nominal": est_ms,
        "allreduce_ms_per_iter_estimate": est_ms / args.interval,
        "note": "one GPU: the AllReduce is skipped (nranks = 1); its time is a nominal-bandwidth estimate "
                "(2(K-1)/K x payload / 900 GB/s), not a measurement",
        "setup_s": round(t_plan, 1),
        "gpu": torch.cuda.get_device_name(0),
    }
    if args.profile:
        from collections import defaultdict

        from torch.profiler import ProfilerActivity, profile

        def kernel_times(fn, n):
            pos[0] = 40
            torch.cuda.synchronize()
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                fn(n)
                torch.cuda.synchronize()
            tot = defaultdict(float)
            iv = []
            for e in prof.events():
                if e.device_type.name == "CUDA":
                    name = e.name.replace("bsg::(anonymous namespace)::", "").replace("void ", "").split("(")[0]
                    tot[name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
                    iv.append((e.time_range.start, e.time_range.end))
            iv.sort()
            busy, cur_s, cur_e = 0.0, None, None
            for a, b in iv:  # union of the kernels' intervals: the GPU's busy time
                if cur_e is None or a > cur_e:
                    if cur_e is not None:
                        busy += cur_e - cur_s
                    cur_s, cur_e = a, b
                else:
                    cur_e = max(cur_e, b)
            if cur_e is not None:
                busy += cur_e - cur_s
            span = (iv[-1][1] - iv[0][0]) if iv else 0.0
            res = {k: round(v / n, 2) for k, v in sorted(tot.items(), key=lambda x: -x[1])}
            res["_busy_us_per_step"] = round(busy / n, 1)
            res["_span_us_per_step"] = round(span / n, 1)
            return res
        out["us_per_step_by_kernel_plain"] = kernel_times(lambda n: [step() for _ in range(n)], 50)
        out["us_per_step_by_kernel_async"] = kernel_times(with_async, 50)
    print(json.dumps(out), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
