"""Summarise one round of GPU evidence into profiles/.

Reads (from gpurun_out/): launches_<tag>.csv (ncu --metrics
gpu__time_duration.sum launch list of `bench.py --profile`) and
full_<kernel>_<tag>.ncu-rep (ncu --set full captures), and writes
  profiles/launches_<tag>.md   per-kernel share of the step (cold-cache, serialised)
  profiles/ncu_<tag>.md        per-kernel SOL, DRAM bytes, pipes, top stalls
  profiles/dram_traffic.json   bench stage -> measured DRAM bytes per step (kernels that run less
                               often than every step scaled by their launches per step)

usage: python tools/profile_summary.py <tag> [gpurun_out]
"""
import collections
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# kernel -> bench stage whose CUDA-event time it dominates
STAGE_OF = {"preprocess_kernel": "preprocess", "blend_fwd_kernel": "blend_fwd", "blend_bwd_kernel": "blend_bwd",
            "adam_kernel": "adam", "adam_rot_kernel": "adam", "adam_sparse_kernel": "adam", "materialize_kernel": "adam", "fold_visible_kernel": "fold", "fold_adam_kernel": "adam", "ssim_windows_kernel": "loss_ssim",
            "ssim_pixels_kernel": "loss_ssim", "onesweep_kernel": "bin_sort", "scan_kernel": "compact",
            "emit_pairs_kernel": "bin_emit", "emit_tiles_kernel": "bin_emit", "tile_sort_kernel": "bin_sort",
            "tile_scan_kernel": "bin_scan", "tile_scan_a_kernel": "bin_scan", "tile_scan_b_kernel": "bin_scan",
            "compact_mask_kernel": "compact"}

METRICS = [
    ("time_us", "gpu__time_duration.sum", 1e-3),
    ("dram_read_MB", "dram__bytes_read.sum", 1e-6),
    ("dram_write_MB", "dram__bytes_write.sum", 1e-6),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("issue_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    ("fma_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("alu_pct", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("xu_pct", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    ("fp64_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("occ_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("grid", "launch__grid_size", 1),
]


def short(name):
    n = name.split("(")[0].replace("(anonymous namespace)::", "").replace("bsg::", "")
    n = n.replace("void ", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    return n.strip()


def base(name):
    return short(name).split("<")[0]


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def launches(path):
    d = collections.defaultdict(list)
    with open(path) as f:
        rows = [r for r in csv.reader(f) if len(r) > 5]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    for r in rows[1:]:
        v = num(r[vi])
        if v is not None:
            d[short(r[ki])].append(v)
    return d


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return None
    h, units, data = rows[0], rows[1], rows[2]
    scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1.0,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = {}
    for k, u, v in zip(h, units, data):
        x = num(v)
        out[k] = x * scale[u] if (x is not None and u in scale) else v
    return out  # times in ns, sizes in bytes


def stalls(m, top=4):
    pre = "smsp__average_warps_issue_stalled_"
    suf = "_per_issue_active.ratio"
    s = [(k[len(pre):-len(suf)], num(v)) for k, v in m.items() if k.startswith(pre) and k.endswith(suf)]
    s = [x for x in s if x[1] is not None]
    s.sort(key=lambda x: -x[1])
    return ", ".join(f"{k} {v:.2f}" for k, v in s[:top])


def main():
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    lp = os.path.join(src, f"launches_{tag}.csv")
    if os.path.exists(lp):
        d = launches(lp)
        tot = sum(sum(v) for v in d.values())
        lines = [f"# Launch list `{tag}` (ncu gpu__time_duration.sum, --clock-control none; cold-cache, serialised)", "",
                 "| kernel | launches | mean us | share of kernel time |", "|---|---|---|---|"]
        for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
            lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / tot:.3f} |")
        lines.append(f"\nTotal kernel time in the capture: {tot / 1e6:.3f} ms")
        open(os.path.join(prof, f"launches_{tag}.md"), "w").write("\n".join(lines) + "\n")
    # launches per step of each kernel (materialize runs every 32 steps): the
    # per-launch DRAM bytes of a capture are scaled to bytes per step
    per_step = {}
    if os.path.exists(lp):
        steps = max((len(v) for k, v in d.items() if base(k) == "preprocess_kernel"), default=0)
        for k, v in d.items():
            if steps:
                per_step[base(k)] = len(v) / steps
    traffic = {}
    tp = os.path.join(prof, "dram_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp))
    kp = os.path.join(prof, "kernel_metrics.json")
    kmet = json.load(open(kp)) if os.path.exists(kp) else {}
    if per_step:  # kernels the current build no longer launches drop out of both files
        traffic = {st: {k: v for k, v in ks.items() if k in per_step} for st, ks in traffic.items()}
        traffic = {st: ks for st, ks in traffic.items() if ks}
        kmet = {k: v for k, v in kmet.items() if k in per_step}
    lines = [f"# ncu --set full captures `{tag}` (one launch each, inside `bench.py --profile`)", "",
             "| kernel | " + " | ".join(k for k, _, _ in METRICS) + " | top stalls (warps per issue) |",
             "|---" * (len(METRICS) + 2) + "|"]
    for rep in sorted(glob.glob(os.path.join(src, f"full_*_{tag}.ncu-rep"))):
        m = raw(rep)
        if not m:
            continue
        name = short(m.get("Kernel Name", os.path.basename(rep)))
        vals = []
        for _, key, sc in METRICS:
            v = num(m.get(key, ""))
            vals.append("NA" if v is None else f"{v * sc:.1f}")
        lines.append(f"| {name} | " + " | ".join(vals) + f" | {stalls(m)} |")
        st = STAGE_OF.get(base(name))
        rd, wr = num(m.get("dram__bytes_read.sum", "")), num(m.get("dram__bytes_write.sum", ""))
        if st and rd is not None and wr is not None:
            traffic.setdefault(st, {})[base(name)] = (rd + wr) * min(1.0, per_step.get(base(name), 1.0))
        kmet[base(name)] = {k: (num(m.get(key, "")) or 0.0) * sc for k, key, sc in METRICS}
        kmet[base(name)]["capture"] = f"profiles/ncu_{tag}.md"
    open(os.path.join(prof, f"ncu_{tag}.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tp, "w"), indent=1, sort_keys=True)
    json.dump(kmet, open(kp, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
