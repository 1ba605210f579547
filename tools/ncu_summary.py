"""Summarise ncu artefacts for profiles/: key metrics of a --set full report and the
per-kernel share of a launch list (gpu__time_duration.sum CSV).

    python tools/ncu_summary.py full REPORT.ncu-rep OUT.csv
    python tools/ncu_summary.py launches LAUNCHES.csv OUT.txt
"""
import csv
import subprocess
import sys
from collections import defaultdict

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "smsp__inst_executed_op_shfl.sum", "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size"]


def full(rep, out):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                       capture_output=True, text=True, check=True)
    rows = list(csv.reader(r.stdout.splitlines()))
    hdr, units = rows[0], rows[1]
    keep = ["Kernel Name"] + [m for m in METRICS if m in hdr]
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(keep)
        w.writerow([""] + [units[hdr.index(m)] for m in keep[1:]])
        for row in rows[2:]:
            w.writerow([row[hdr.index(k)] for k in keep])


def launches(path, out):
    agg = defaultdict(lambda: [0, 0.0])
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            try:
                v = float(d["Metric Value"].replace(",", ""))
            except ValueError:
                continue
            unit = d.get("Metric Unit", "ns")
            v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
            k = d["Kernel Name"].split("(")[0]
            agg[k][0] += 1
            agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'ms/launch':>10s} {'share':>6s}\n")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{k:40s} {v[0]:8d} {v[1]:10.3f} {v[1] / v[0]:10.3f} {100 * v[1] / tot:5.1f}%\n")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
