"""Per-instruction execution counts of one kernel from an ncu --set full
report (source page, SASS view): prints the SASS with warp-level execution
counts and the share of the kernel's issued instructions, so hot loops can be
read instruction by instruction.

usage: python tools/sass_hot.py <report.ncu-rep> [--min-share 0.002] [--range a:b]
"""
import argparse
import csv
import io
import subprocess


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc, iexe, ithr = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), \
        hdr.index("Thread Instructions Executed")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    res = []
    for r in rows[2:]:
        if len(r) <= iexe:
            continue
        try:
            res.append((r[ia], r[isrc].strip(), int(r[iexe] or 0), int(r[ithr] or 0), int(r[isamp] or 0)))
        except ValueError:
            continue
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--min-share", type=float, default=0.0)
    ap.add_argument("--range", default=None)
    a = ap.parse_args()
    rows = load(a.rep)
    tot = sum(r[2] for r in rows)
    stot = sum(r[4] for r in rows) or 1
    lo, hi = (0, len(rows))
    if a.range:
        lo, hi = (int(x) for x in a.range.split(":"))
    print(f"total warp instructions {tot}")
    for k, (addr, src, exe, thr, samp) in enumerate(rows[lo:hi], lo):
        if exe / max(tot, 1) >= a.min_share:
            act = thr / exe if exe else 0
            print(f"{k:4d} {exe:10d} {100 * exe / tot:5.2f}% act{act:5.1f} st{100 * samp / stot:5.2f}%  {src}")


if __name__ == "__main__":
    main()
