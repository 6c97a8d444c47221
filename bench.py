"""Benchmark of the DOGS block-training hot path on B200.

Headline workload (BASELINE.json configs[2], SURVEY §8(d) cfg 3 -- the
largest configuration named for the 8xB200 box, run at K = N blocks):
synthetic large aerial scene, 6M Gaussians in a 100 x 20 x 100 box, 96 views
at 1600x1066 on a jittered aerial grid 5 degrees off nadir, K = N blocks (one
per GPU, recursive longer-axis split with expansion s = 1.4, consensus every
`interval` iterations). A step is one training iteration of every block
(projection, binning, render fwd, L1+SSIM loss, render bwd, fold, ADMM
penalty + Adam) plus the amortised consensus round. Ground truth is rendered
once by the device forward from the generating cloud; training starts from a
perturbed copy. The view order is BlockTrainer's (trainer.cpp:250-252), so
the reference arm replays the same views.

At N = 1 the same JSON line also carries (under "also") cfg 2 (configs[1]:
2M Gaussians, 1024x768, 64 views) at the bench's 5 degree tilt and at 30
degrees (the camera plane cuts the scene slab: near-plane splats cover whole
views), and the consensus round of block 0 of cfg 3's K = 8 plan on this GPU.

`--impl reference` times the reference's CPU algorithm (the oracle port,
oracle/_oracle: FP64 BlockTrainer::train_step, one thread per block as the
reference runs, runtime.cpp:641-666) on the same block, view order and
ground truth (rendered by the oracle's own FP64 renderer), on rank 0.
"""
import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
CFGS = {
    "cfg2": dict(n=2_000_000, width=1024, height=768, views=64, extent=100.0, scale=1.4, seed=42, tilt=5.0),
    "cfg2_tilt30": dict(n=2_000_000, width=1024, height=768, views=64, extent=100.0, scale=1.4, seed=42, tilt=30.0),
    "cfg3": dict(n=6_000_000, width=1600, height=1066, views=96, extent=100.0, scale=1.4, seed=42, tilt=5.0),
    "cfg4": dict(n=20_000_000, width=1600, height=1066, views=96, extent=100.0, scale=2.0, seed=42, tilt=5.0),
}
WORKLOAD = {
    "cfg2": "cfg2 (configs[1]): 2M Gaussians, 64 views 1024x768, 5 deg off nadir",
    "cfg2_tilt30": "cfg2 geometry at 30 deg off nadir (near-plane splats cover whole views)",
    "cfg3": "cfg3 (configs[2]): 6M Gaussians, 96 views 1600x1066, 5 deg off nadir",
    "cfg4": "cfg4 (configs[3]): 20M Gaussians, K=8 at s=2.0 (high shared overlap), 1600x1066 views",
}
TRAIN_SEED = 1  # TrainerConfig::seed of both arms (view order)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="cfg3", choices=sorted(CFGS))
    p.add_argument("--interval", type=int, default=25, help="consensus interval (iterations)")
    p.add_argument("--gaussians", type=int, default=None, help="override the Gaussian count (profiling, tests)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-also", action="store_true", help="skip the secondary configurations")
    p.add_argument("--views", type=int, default=None, help="fewer views for profiling runs only")
    p.add_argument("--profile", action="store_true",
                   help="ncu mode: constant ground truth (no GT renders), no e2e/CPU/secondary legs")
    return p.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    try:
        with open(MEASURED_PEAKS) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled through NVML every ~1 ms from a
    background thread; stop(t0, t1) keeps the samples inside [t0, t1] (the
    timed region). Falls back to `nvidia-smi -lms 20` without NVML."""

    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20), ("hw_thermal_slowdown", 0x40),
               ("hw_power_brake_slowdown", 0x80), ("sw_power_cap", 0x4))

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.run = False
        self.h = None
        self.max_mhz = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.h = None
            return self._start_smi()
        self.run = True
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()

    def _poll(self):
        nv = self.nv
        while self.run:
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                break
            self.samples.append((time.perf_counter(), float(mhz), int(rs)))
            time.sleep(0.001)

    def _start_smi(self):
        import subprocess
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={fields}",
                                          "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def read():
            names = [0x8, 0x40, 0x20, 0x4]
            for line in self.proc.stdout:
                parts = [x.strip() for x in line.split(",")]
                try:
                    rs = sum(b for b, v in zip(names, parts[2:6]) if v.lower() == "active")
                    self.max_mhz = float(parts[1])
                    self.samples.append((time.perf_counter(), float(parts[0]), rs))
                except (ValueError, IndexError):
                    continue
        self.t = threading.Thread(target=read, daemon=True)
        self.t.start()

    def wait_first(self, timeout=5.0):
        t = time.perf_counter()
        while not self.samples and time.perf_counter() - t < timeout:
            time.sleep(0.005)

    def window(self, t0, t1):
        sm, reasons = [], set()
        for ts, mhz, rs in self.samples:
            if t0 <= ts <= t1:
                sm.append(mhz)
                for nm, bit in self.REASONS:
                    if rs & bit:
                        reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvml" if self.h else "nvidia-smi"}

    def stop(self):
        self.run = False
        if getattr(self, "proc", None):
            self.proc.terminate()


# ---------------------------------------------------------------- scene ---

def scene(cfg, n=None):
    from paper_2405_13943_b200.scene import aerial_scene, perturbed_init
    cloud, cams = aerial_scene(n or cfg["n"], cfg["width"], cfg["height"], cfg["views"], cfg["extent"], cfg["seed"],
                               tilt_deg=cfg["tilt"])
    return cloud, cams, perturbed_init(cloud, cfg["seed"])


def build_block(cfg, rank, world, device, n=None, n_views=None, constant_gt=False):
    """Scene -> plan -> this rank's block on the device, GT rendered on device."""
    from paper_2405_13943_b200 import api

    cloud, cams, init = scene(cfg, n)
    centers = np.array([c.center() for c in cams])
    plan = api.Plan(cloud["ids"], cloud["pos"], centers, world, cfg["scale"])
    ids, views = plan.block(rank)
    if n_views:
        views = views[:n_views]
    sel = ids.astype(np.int64)  # ids are 0..n-1 = row indices of the global cloud
    view_cams = [cams[v].device() for v in views]
    if constant_gt:
        gts = [np.full((cfg["height"], cfg["width"], 3), 0.5) for _ in view_cams]
    else:
        gt_block = api.Block(device, 3)
        gt_block.upload_cloud(cloud["ids"], cloud["pos"], cloud["rot"], cloud["ls"], cloud["feat"], cloud["op"])
        gts = [gt_block.render(c)[0] for c in view_cams]
        gt_block.close()
    blk = api.Block(device, 3)
    blk.upload_cloud(init["ids"][sel], init["pos"][sel], init["rot"][sel], init["ls"][sel], init["feat"][sel],
                     init["op"][sel])
    blk.set_views(view_cams, gts)
    blk.trainer_init(api.trainer_config(iterations=30000, densify={"enabled": 0}))
    sids, cnt, _ = plan.shared()
    rows, slots, first = plan.block_shared(rank)
    if world > 1:
        blk.set_shared(rows, slots, first, cnt)
        init_rows = np.concatenate([init["pos"], init["rot"], init["ls"], init["feat"], init["op"][:, None]], 1)
        zprev = init_rows[sids.astype(np.int64)]
        blk.set_anchor(zprev[slots], zprev, api.penalties())
    info = dict(block_gaussians=len(ids), block_views=len(views), shared_ids=len(sids), block_shared=len(rows))
    return blk, view_cams, gts, info


STAGE_KERNEL = {"blend_bwd": "blend_bwd_kernel", "blend_fwd": "blend_fwd_kernel", "adam": "fold_adam_kernel",
                "preprocess": "preprocess_kernel", "loss_ssim": "ssim_windows_kernel"}


def algorithmic_bytes(stage, n, V, P, HW, shared):
    """SURVEY §8(d) fused-minimum byte accounting per launch of each stage
    (n rows, V visible splats, P tile pairs, HW pixels, D = 14 FP32 components
    per row at SH degree 0). DESIGN.md §3 lists the same figures."""
    D4 = 56
    model = {
        # fold + lazy Adam, one kernel: the visible row's 2D gradient record read, its x, m, v
        # read + written once; every row caught up once per 16 steps (x, m, v read + written, stamp); shared
        # rows: x, m, v, z, u (the penalty keeps them current every step)
        "adam": (48 + 6 * D4 + 8) * V + (6 * D4 + 4) * n // 16 + 8 * D4 * shared,
        # pos + log-scale + step stamp of every row, tiles-touched and the visibility bit written; rest of the
        # row, splat record, depth key, zeroed gradient record for visible rows
        "preprocess": 32 * n + n // 8 + (32 + 48 + 8 + 48) * V,
        # per-tile path: the visibility mask read, the visible rows written
        "compact": n // 8 + 4 * V,
        # per-tile binning (the path taken at this config):
        "bin_scan": 0,                              # tile scan: a few KB of per-tile counts / ranges
        "bin_emit": 4 * V + 16 * V + 4 * P,         # visible row + its rect read, one row written per pair
        "bin_sort": 4 * P + 8 * P + 4 * P,          # rows read, their FP64 depth gathered, sorted rows written
        "blend_fwd": 52 * P + 24 * HW,              # pair row + 48 B record per pair; rgb, T, n, last per pixel
        "loss_ssim": 36 * HW,                       # rendered + GT read, dL/dC written (fused minimum)
        "blend_bwd": 52 * P + 20 * HW + 48 * V,     # records; T, last, dL/dC per pixel; one gradient record per splat
    }
    return model.get(stage)


class Runner:
    """Steps of one block in BlockTrainer's view order, with optional
    asynchronous consensus rounds every `interval` iterations."""

    def __init__(self, blk, n_views, rank, world, interval):
        from paper_2405_13943_b200 import api
        self.blk, self.world, self.interval = blk, world, interval
        self.seq = [int(v) for v in api.view_sequence(TRAIN_SEED, rank, n_views, 200000)]
        self.pos, self.it, self.pending = 0, 0, False
        self.round_ms = []

    def next_view(self):
        v = self.seq[self.pos % len(self.seq)]
        self.pos += 1
        return v

    def consensus(self, flush=False, on=True):
        """a round every `interval` iterations, asynchronous; it
        overlaps the next step's projection/sort/blends/fold, only that step's
        Adam waits; its result is collected after the next step is enqueued."""
        if self.pending:
            self.round_ms.append(self.blk.consensus_wait()["ms"])
            self.pending = False
        if on and self.world > 1 and not flush and self.it % self.interval == 0:
            self.blk.consensus_round_async(1.6, True, iteration=self.it)
            self.pending = True

    def steps(self, k, consensus=True):
        for _ in range(k):
            self.blk.train_steps([self.next_view()], want_losses=False)
            self.it += 1
            self.consensus(on=consensus)


def timed_region(run, stream, k, world, consensus=True):
    """Barrier + synchronize, k steps between CUDA events on the block's
    stream, synchronize + barrier; max over ranks. Returns ms per step."""
    import torch
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tc0 = time.perf_counter()
    e0.record(stream)
    run.steps(k, consensus)
    run.consensus(flush=True)
    e1.record(stream)
    torch.cuda.synchronize()
    tc1 = time.perf_counter()
    barrier(world)
    return max_over_ranks(e0.elapsed_time(e1), world) / k, tc0, tc1


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world):
    import torch
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([float(v)], device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return float(v)


def host_allreduce(arr, op):
    """The host communicator's reduction over the process group (ranks that
    share a GPU cannot share an NCCL communicator)."""
    import torch
    import torch.distributed as dist
    dist.all_reduce(torch.from_numpy(arr), op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)


def stage_pass(run, steps):
    blk = run.blk
    blk.enable_stage_timing(True)
    acc, cnt = {}, dict(visible=0, pairs=0, blend_evals=0)
    for _ in range(steps):
        run.steps(1)
        for k, v in blk.stage_times().items():
            acc[k] = acc.get(k, 0.0) + v
        c = blk.step_counters()
        for k in cnt:
            cnt[k] += c[k]
    run.consensus(flush=True)
    blk.enable_stage_timing(False)
    return {k: v / steps for k, v in acc.items()}, {k: v / steps for k, v in cnt.items()}


def secondary(name, device, steps, warmup):
    """One extra configuration at N = 1: ms/step and the stage split."""
    import torch
    cfg = CFGS[name]
    t0 = time.time()
    blk, cams, _, info = build_block(cfg, 0, 1, device)
    run = Runner(blk, len(cams), 0, 1, 25)
    stream = torch.cuda.ExternalStream(blk.stream())
    run.steps(warmup)
    ms, _, _ = timed_region(run, stream, steps, 1)
    stage, cnt = stage_pass(run, min(steps, 50))
    blk.close()
    return {"workload": WORKLOAD[name], "value": 1000.0 / ms, "unit": "iters/s", "ms_per_step": ms,
            "steps": steps, "gaussians": cfg["n"], "width": cfg["width"], "height": cfg["height"],
            "tilt_deg": cfg["tilt"], "visible_per_step": cnt["visible"], "pairs_per_step": cnt["pairs"],
            "stage_ms": {k: round(v, 4) for k, v in stage.items()}, "wall_s": round(time.time() - t0, 1)}


def consensus_k8(device, name="cfg3", steps=100, interval=25):
    """ADMM consensus ms/iter (BASELINE metric) of the K = 8 plan of cfg 3
    (or cfg 4: s = 2.0, the consensus stress) on one GPU: block 0 with its
    real shared set and slot table; the round's device work (sign pre-pass,
    relaxed pack, unpack / duals / residuals, device penalty adaptation)
    measured, asynchronous, against the same steps without rounds. One rank,
    so the all-reduce itself is not on the wire; its payload is reported with
    a nominal NVLink 5 time."""
    import torch

    from paper_2405_13943_b200 import api
    cfg = CFGS[name]
    cloud, cams, init = scene(cfg)
    centers = np.array([c.center() for c in cams])
    plan = api.Plan(cloud["ids"], cloud["pos"], centers, 8, cfg["scale"])
    ids, views = plan.block(0)
    sids, cnt, _ = plan.shared()
    rows, slots, first = plan.block_shared(0)
    sel = ids.astype(np.int64)
    blk = api.Block(device, 3)
    blk.upload_cloud(init["ids"][sel], init["pos"][sel], init["rot"][sel], init["ls"][sel], init["feat"][sel],
                     init["op"][sel])
    vcams = [cams[v].device() for v in views]
    blk.set_views(vcams, [np.full((cfg["height"], cfg["width"], 3), 0.5) for _ in vcams])
    blk.trainer_init(api.trainer_config(iterations=30000, densify={"enabled": 0}))
    # one rank holds only its own contribution: one owner per slot keeps its z
    # (and so the training cost) undisturbed; same kernels and sizes
    blk.set_shared(rows, slots, np.ones_like(first), np.ones_like(cnt))
    init_rows = np.concatenate([init["pos"], init["rot"], init["ls"], init["feat"], init["op"][:, None]], 1)
    zprev = init_rows[sids.astype(np.int64)]
    blk.set_anchor(zprev[slots], zprev, api.penalties())
    del cloud, init, init_rows
    stream = torch.cuda.ExternalStream(blk.stream())
    run = Runner(blk, len(vcams), 0, 2, interval)  # world 2: rounds on; the block's communicator is local
    run.steps(10, consensus=False)
    for _ in range(2):
        blk.consensus_round_async(1.6, True, iteration=0)
        run.steps(1, consensus=False)
        blk.consensus_wait()
    # Windows of `interval` steps, alternately without and with a round at
    # their start (waited after the window's first step, as in training): the
    # model keeps training, so interleaving keeps both sides on the same state
    # (timing all plain steps first and all rounds after measured the drift of
    # the step cost as consensus overhead).
    rounds, t_plain, t_round = [], 0.0, 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    windows = max(1, steps // interval)
    vs = []
    for w in range(2 * windows):
        with_round = w % 2 == 1
        if not with_round:  # both windows of a pair render the same views (the step cost is view-dependent)
            vs = [run.next_view() for _ in range(interval)]
        torch.cuda.synchronize()
        e0.record(stream)
        if with_round:
            blk.consensus_round_async(1.6, True, iteration=run.it)
        for j in range(interval):
            blk.train_steps([vs[j]], want_losses=False)
            run.it += 1
            if with_round and j == 0:
                rounds.append(blk.consensus_wait()["ms"])
        e1.record(stream)
        torch.cuda.synchronize()
        if with_round:
            t_round += e0.elapsed_time(e1)
        else:
            t_plain += e0.elapsed_time(e1)
    plain = t_plain / (windows * interval)
    with_async = t_round / (windows * interval)
    blk.close()
    D, S, K = 14, len(sids), 8
    payload = 4 * 4 * S + 4 * (D + 1) * S + 8 * 3
    est = 2 * (K - 1) / K * payload / 900e9 * 1e3
    rms = float(np.mean(rounds)) if rounds else None
    return {"workload": "%s K=8 plan (s=%.1f), block 0 on this GPU (its real shared set), interval %d" %
                        (name, cfg["scale"], interval),
            "block0_gaussians": int(len(ids)), "block0_shared_rows": int(len(rows)), "global_shared_slots": int(S),
            "round_ms_device": rms, "consensus_ms_per_iter": (rms / interval) if rms else None,
            "ms_per_step_no_rounds": plain, "ms_per_step_async_rounds": with_async,
            "consensus_ms_per_iter_exposed": with_async - plain,
            "comm_fraction": ((rms / interval) / with_async) if rms else None,
            "allreduce_bytes_per_round": payload, "allreduce_ms_nvlink5_nominal": est,
            "note": "one GPU: the round's kernels are measured; the all-reduce of allreduce_bytes_per_round over "
                    "NVLink is the nominal-bandwidth estimate (2(K-1)/K x bytes / 900 GB/s), not a measurement"}


# ------------------------------------------------------------- our arm ---

def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2405_13943_b200 import api

    cfg = CFGS[args.config]
    ndev = torch.cuda.device_count()
    device = local_rank % ndev
    shared_gpu = world > ndev  # more ranks than GPUs (a test of the N > 1 flow on one GPU)
    torch.cuda.set_device(device)
    if world > 1:
        import torch.distributed as dist
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
    blk, view_cams, gts, info = build_block(cfg, rank, world, device, args.gaussians, args.views, args.profile)
    if world > 1:
        import torch.distributed as dist
        if shared_gpu:
            blk.comm_init_host(host_allreduce, world, rank)
        else:
            uid = [api.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            blk.comm_init(uid[0], world, rank)
        blk.set_round_timeout(120.0)
    nv = len(view_cams)
    run = Runner(blk, nv, rank, world, args.interval)
    stream = torch.cuda.ExternalStream(blk.stream())
    clocks = ClockSampler(device)
    clocks.start()
    clocks.wait_first()
    run.steps(args.warmup)
    run.consensus(flush=True)
    launches0 = blk.launch_count()
    ms_step, tc0, tc1 = timed_region(run, stream, args.steps, world)
    launches = blk.launch_count() - launches0
    clk = clocks.window(tc0, tc1)
    round_ms = list(run.round_ms)
    # multi-GPU: the same steps without rounds, for the exposed consensus cost
    ms_plain = None
    if world > 1:
        ms_plain, _, _ = timed_region(run, stream, args.steps, world, consensus=False)
    stage_ms, cnt = stage_pass(run, min(args.steps, 100))
    if args.profile:
        clocks.stop()
        if rank == 0:
            print(json.dumps({"profile_run": True, "ms_per_step": ms_step}), flush=True)
        return
    # end-to-end through bsg_train_steps_host_u8: every step's ground truth as
    # the 8-bit RGB the reference trains from (its images are PPM bytes,
    # image.cpp:60-79; the rendered GT is quantized once, image.cpp:12-19)
    # copied from pinned host memory, every step's loss read back
    pinned = [torch.from_numpy(np.clip(np.rint(np.clip(g, 0.0, 1.0) * 255.0), 0, 255).astype(np.uint8)).pin_memory()
              for g in gts]
    del gts
    e2e_steps = max(5, args.steps)
    for _ in range(max(1, min(args.warmup, 5))):
        v = run.next_view()
        blk.train_steps_host_u8([view_cams[v]], [pinned[v].numpy()])
        run.it += 1
        run.consensus()
    run.consensus(flush=True)
    barrier(world)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    done = 0
    while done < e2e_steps:
        # up to the next consensus point: one host-image call (the GT of every
        # step uploaded from pinned memory on a copy stream, double-buffered,
        # while the previous step computes; every step's loss read back)
        k = min(args.interval - run.it % args.interval, e2e_steps - done)
        vs = [run.next_view() for _ in range(k)]
        blk.train_steps_host_u8([view_cams[v] for v in vs], [pinned[v].numpy() for v in vs])
        run.it += k
        done += k
        run.consensus()
    run.consensus(flush=True)
    f1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    e2e_ms_step = max_over_ranks(f0.elapsed_time(f1), world) / e2e_steps
    h2d = 3 * cfg["width"] * cfg["height"]  # 8-bit RGB per step
    clocks.stop()

    if rank != 0:
        blk.close()
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    V, P, HW = cnt["visible"], cnt["pairs"], cfg["width"] * cfg["height"]
    nb = info["block_gaussians"]
    peak, peak_kind = peaks()
    traffic_all = {}
    prof = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(prof):
        try:
            traffic_all = json.load(open(prof))
        except Exception:
            traffic_all = {}

    def roof(stage):
        b = algorithmic_bytes(stage, nb, V, P, HW, info["block_shared"])
        if not b or stage_ms.get(stage, 0) <= 0:
            return None
        a = b / (stage_ms[stage] * 1e-3) / 1e9
        tr = traffic_all.get(stage)
        return {"kernel": stage, "bound": "hbm", "achieved": a, "peak": peak, "unit": "GB/s", "frac": a / peak,
                "traffic": float(sum(tr.values())) if tr else None, "algorithmic_bytes_per_launch": b,
                "peak_source": peak_kind}

    stage_roofs = {k: roof(k) for k in stage_ms if roof(k) is not None}
    roof_stage = max(stage_roofs, key=lambda k: stage_ms[k])
    roofline = stage_roofs[roof_stage]
    kmet_path = os.path.join(ROOT, "profiles", "kernel_metrics.json")
    if os.path.exists(kmet_path):
        try:
            km = json.load(open(kmet_path)).get(STAGE_KERNEL.get(roof_stage, ""), None)
        except Exception:
            km = None
        if km:
            roofline["compute"] = {"bound": "sm_issue", "issue_slots_busy_pct": round(km["issue_pct"], 1),
                                   "fma_pipe_pct": round(km["fma_pct"], 1), "alu_pipe_pct": round(km["alu_pct"], 1),
                                   "xu_pipe_pct": round(km["xu_pct"], 1), "source": km["capture"]}
    # useful FP32 work of the blends: per composited (pixel, contributor)
    # pair ~15 FLOP + 1 exp forward, ~40 FLOP + 1 exp + 1 reciprocal backward
    evals = cnt["blend_evals"]
    sm_mhz = clk.get("sm_mhz") or 1965.0
    fp32_peak = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12
    mufu_peak = 148 * 16 * sm_mhz * 1e6 / 1e12
    blend_work = {}
    for st, flop, mufu in (("blend_fwd", 15, 1), ("blend_bwd", 40, 2)):
        if stage_ms.get(st):
            t = stage_ms[st] * 1e-3
            blend_work[st] = {"evaluations": evals, "tflops": evals * flop / t / 1e12,
                              "fp32_frac": evals * flop / t / 1e12 / fp32_peak,
                              "mufu_frac": evals * mufu / t / 1e12 / mufu_peak}
    if roof_stage in blend_work:
        roofline.setdefault("compute", {}).update({"fp32_tflops": round(blend_work[roof_stage]["tflops"], 3),
                                                   "fp32_peak_tflops": round(fp32_peak, 1),
                                                   "fp32_frac": round(blend_work[roof_stage]["fp32_frac"], 4),
                                                   "mufu_frac": round(blend_work[roof_stage]["mufu_frac"], 4)})
    rms = float(np.mean(round_ms)) if round_ms else None
    out = {
        "metric": "training iters/sec (K=N blocks, 1 block per GPU)",
        "value": 1000.0 / ms_step,
        "unit": "iters/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32 (FP64 projection)",
        "data": "synthetic (aerial scene, GT rendered on device from the generating cloud; training from a "
                "perturbed copy)",
        "config": {"workload": WORKLOAD[args.config] + (f" ({args.gaussians} Gaussians)" if args.gaussians else ""),
                   "gaussians": args.gaussians or cfg["n"], "width": cfg["width"], "height": cfg["height"],
                   "views": cfg["views"], "tilt_deg": cfg["tilt"], "blocks": world, "expand_scale": cfg["scale"],
                   "consensus_interval": args.interval, "block0_gaussians": nb, "block0_views": info["block_views"],
                   "shared_ids": info["shared_ids"], "view_order": "BlockTrainer (trainer.cpp:250-252), seed 1",
                   "l2": "inputs > L2 (Adam state %.1fM rows x 168 B)" % (nb / 1e6),
                   "parallelism": f"blocks{world}",
                   "transport": ("nccl" if not shared_gpu else "host all-reduce over gloo (ranks share a GPU)")
                   if world > 1 else None},
        "e2e": {"value": 1000.0 / e2e_ms_step, "unit": "iters/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 24},
        "e2e_path": "bsg_train_steps_host_u8: every step's 8-bit RGB ground truth (the reference's PPM data, quantized "
                    "once) copied from pinned host memory and widened on the device; every step's loss read back",
        # value = global iterations/s (Alg. 2: one local step of every block); each GPU trains its own
        # block on one view per iteration, so the job's block-step throughput is K x value
        "block_steps_per_s": world * 1000.0 / ms_step,
        "gpu_launches": int(launches),
        "stage_ms": {k: round(v, 4) for k, v in stage_ms.items()},
        "stage_ms_note": "separate pass with CUDA events between stages (adds one host sync per step)",
        "dominant_stage": max(stage_ms, key=stage_ms.get),
        "visible_per_step": V,
        "blend_evaluations_per_step": evals,
        "blend_work": blend_work,
        "pairs_per_step": P,
        "consensus_ms_per_round": rms or 0.0,
        "consensus_ms_per_iter": (rms / args.interval) if rms else 0.0,
        "roofline": roofline,
        "stage_rooflines": {k: {"achieved": round(v["achieved"], 1), "frac": round(v["frac"], 4),
                                "algorithmic_bytes": round(v["algorithmic_bytes_per_launch"]),
                                "traffic": v["traffic"]} for k, v in stage_roofs.items()},
        "clocks": clk,
    }
    if world > 1:
        out["consensus"] = {"round_ms_device": rms, "ms_per_step_no_rounds": ms_plain,
                            "consensus_ms_per_iter_exposed": ms_step - ms_plain,
                            "comm_fraction": ((rms / args.interval) / ms_step) if rms else None,
                            "exposed_fraction": (ms_step - ms_plain) / ms_step}
    blk.close()
    del pinned
    if world == 1 and not args.no_also:
        also = {}
        for name in ("cfg2", "cfg2_tilt30"):
            if name != args.config:
                also[name] = secondary(name, device, max(args.steps, 100), max(args.warmup, 5))
        also["consensus_k8"] = consensus_k8(device, "cfg3")
        also["consensus_cfg4_k8"] = consensus_k8(device, "cfg4")
        out["also"] = also
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, args.gaussians)
    print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ------------------------------------------------------- reference arm ---

def oracle_block(cfg, n, n_gt_views):
    """The reference algorithm on the same block (K=1 at N=1): the FP64 CPU
    BlockTrainer on the perturbed cloud, views in BlockTrainer's order, ground
    truth rendered from the generating cloud by the oracle's FP64 renderer for
    the first n_gt_views views of that order (the others are never reached)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import _oracle as orc
    from concurrent.futures import ThreadPoolExecutor

    cloud, cams, init = scene(cfg, n)

    def ocam(c):
        o = orc.Camera()
        o.fx, o.fy, o.cx, o.cy = c.fx, c.fy, c.cx, c.cy
        o.set_rotation_quat(list(c.q))
        o.t = list(c.t)
        o.width, o.height = c.width, c.height
        return o

    cs = [ocam(c) for c in cams]
    seq = list(orc.view_sequence(TRAIN_SEED, 0, len(cs), n_gt_views))
    gen = orc.Cloud(cloud["ids"], cloud["pos"], cloud["rot"], cloud["ls"], cloud["feat"], cloud["op"])
    del cloud
    blank = np.zeros((cfg["height"], cfg["width"], 3))
    need = sorted(set(seq))
    with ThreadPoolExecutor(max_workers=min(len(need), os.cpu_count() or 1)) as ex:
        rendered = dict(zip(need, ex.map(lambda v: orc.render(gen, cs[v], orc.RenderConfig())[0], need)))
    del gen
    gt = [rendered.get(v, blank) for v in range(len(cs))]
    oc = orc.Cloud(init["ids"], init["pos"], init["rot"], init["ls"], init["feat"], init["op"])
    tc = orc.TrainerConfig()
    tc.iterations, tc.seed = 30000, TRAIN_SEED
    tc.densify_enabled = False
    return orc.BlockTrainer(0, oc, cs, gt, [], n or cfg["n"], tc)


def cpu_baseline(cfg, n, steps=2):
    t0 = time.time()
    tr = oracle_block(cfg, n, steps + 1)
    setup = time.time() - t0
    tr.train_step()  # warm-up (first-touch page faults of the FP64 state)
    t0 = time.perf_counter()
    for _ in range(steps):
        tr.train_step()
    dt = time.perf_counter() - t0
    return {"value": steps / dt, "unit": "iters/s", "cores": 1, "kind": "port",
            "sample": f"{steps} FP64 train_step()s (after 1 warm-up) of the full block ({n or cfg['n']} Gaussians, "
                      f"{cfg['width']}x{cfg['height']}, BlockTrainer view order, oracle-rendered GT) by the oracle "
                      f"port built -O3, one thread as the reference runs one thread per block; {dt:.1f} s "
                      f"(+{setup:.0f} s setup)"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = CFGS[args.config]
    budget = 150.0  # seconds of timed FP64 steps (one step of cfg 3 takes ~10-15 s)
    warm = min(args.warmup, 2)
    est_steps = min(args.steps, 16)
    tr = oracle_block(cfg, args.gaussians, warm + est_steps)
    for _ in range(warm):
        tr.train_step()
    t0 = time.perf_counter()
    done = 0
    for _ in range(args.steps):
        tr.train_step()
        done += 1
        if time.perf_counter() - t0 > budget or done >= est_steps:
            break
    dt = time.perf_counter() - t0
    v = done / dt
    out = {"metric": "training iters/sec (K=N blocks, 1 block per GPU)", "value": v, "unit": "iters/s",
           "n_gpus": world, "steps": done, "warmup": warm, "ms_per_step": 1000.0 * dt / done,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "impl": "reference",
           "data": "synthetic (the same scene, block, view order; GT rendered from the generating cloud by the "
                   "reference's FP64 renderer)",
           "config": {"workload": WORKLOAD[args.config] + " -- block 0 (K=1)" + (f" ({args.gaussians} Gaussians)" if args.gaussians else ""),
                      "gaussians": args.gaussians or cfg["n"], "width": cfg["width"], "height": cfg["height"],
                      "views": cfg["views"], "tilt_deg": cfg["tilt"], "blocks": 1,
                      "view_order": "BlockTrainer (trainer.cpp:250-252), seed 1"},
           "cpu_baseline": {"value": v, "unit": "iters/s", "cores": 1, "kind": "port",
                            "sample": f"{done} train_step()s after {warm} warm-up(s) (capped at {est_steps} steps / "
                                      f"{budget:.0f} s: an FP64 step of this block takes seconds), oracle port of "
                                      f"the reference BlockTrainer built -O3, one thread (one per block, "
                                      f"runtime.cpp:641-666)"},
           "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
