"""Summarise ncu captures into profiles/: per-kernel launch list shares (from the
`--metrics gpu__time_duration.sum` pass) and the key metrics of the `--set full` captures.

    python tools/profile_summary.py gpurun_out/launches.csv gpurun_out/edge_full.ncu-rep \
        gpurun_out/las_full.ncu-rep > profiles/rNN_summary.md
"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            v *= {"ms": 1000.0, "us": 1.0, "ns": 1e-3, "s": 1e6}.get(d["Metric Unit"], 1.0)
            k = d["Kernel Name"].split("(")[0][:60]
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += v
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"## Launch list ({path}; cold-cache, serialised under ncu)\n")
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
        print(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
    print()


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print(f"## `{d.get('Kernel Name', '?')[:100]}` ({path}, ncu --set full)\n")
        print("| metric | value |\n|---|---|")
        for key, label in KEYS:
            if key in d:
                print(f"| {label} (`{key}`) | {d[key]} {u.get(key, '')} |")
        print()


if __name__ == "__main__":
    for p in sys.argv[1:]:
        if p.endswith(".csv"):
            launches(p)
        else:
            full(p)
