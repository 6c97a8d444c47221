import csv, subprocess, sys
def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, data = rows[0], rows[1], rows[2:]
    want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
            'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
            'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
            'launch__grid_size', 'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct']
    idx = [h.index(w) if w in h else -1 for w in want]
    for r in data:
        name = r[idx[0]].split('(')[0].replace('(anonymous namespace)::', '').replace('bsg::', '')[-40:]
        vals = [(r[i] + ' ' + units[i]) if i >= 0 else 'NA' for i in idx[1:]]
        print(f"{name:40s} | " + ' | '.join(v[:22] for v in vals))
for rep in sys.argv[1:]:
    summary(rep)
