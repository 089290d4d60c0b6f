"""Writes a text summary of an ncu launch list (--metrics gpu__time_duration)
and of one `ncu --set full` report into profiles/.
usage: summarize_ncu.py launches.csv full.ncu-rep out.txt [title]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = [f"{'launches':>8} {'avg_ns':>12} {'share':>7}  kernel"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{len(v):8d} {sum(v) / len(v):12.1f} {sum(v) / tot:7.1%}  {k[:110]}")
    return out


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = []
    for d in rows[2:]:
        out.append(f"kernel: {d[h.index('Kernel Name')][:120]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"  {k} = {d[i]} {u[i]}")
    return out


if __name__ == "__main__":
    lines = [f"# {sys.argv[4] if len(sys.argv) > 4 else 'ncu summary'}", "", "## launch list (ncu gpu__time_duration, cold-cache, serialised)"]
    lines += launches(sys.argv[1])
    lines += ["", "## ncu --set full (one launch)"]
    lines += full(sys.argv[2])
    open(sys.argv[3], "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
