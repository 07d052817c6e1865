"""Turns the ncu captures in gpurun_out/ into committed summaries under profiles/:
  profiles/ncu_traffic.json        DRAM bytes (read+write) per launch, per config and kernel
  profiles/r01_ncu_c2_full.csv     key metrics of the C2 full capture
  profiles/r01_launches_bench_c2.csv  the launch list of `python bench.py` (C2)
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
G = ROOT / "gpurun_out"
P = ROOT / "profiles"


def short(name):
    for k in ("bucket_hist", "bucket_colscan", "bucket_partition", "bucket_sort", "bucket_bitset",
              "scatter_kernel", "scan_kernel", "scan2_kernel", "tile_count", "tile_offsets", "key_max"):
        if k in name:
            return {"scatter_kernel": "bitset_scatter", "scan_kernel": "bitset_scan",
                    "scan2_kernel": "bitset_scan"}.get(k, k)
    return name[:40]


def rows(path):
    lines = [l for l in Path(path).read_text().splitlines() if l.startswith('"')]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


traffic = json.loads((P / "ncu_traffic.json").read_text()) if (P / "ncu_traffic.json").exists() else {}
for cfg in ("C3", "C4", "C5"):
    f = G / f"traffic_{cfg}.csv"
    if not f.exists():
        continue
    acc = defaultdict(lambda: defaultdict(list))
    for r in rows(f):
        acc[short(r["Kernel Name"])][r["Metric Name"]].append(float(r["Metric Value"].replace(",", "")))
    out = {}
    for k, m in acc.items():
        rd = m.get("dram__bytes_read.sum", [])
        wr = m.get("dram__bytes_write.sum", [])
        # ncu reports bytes in the unit column; values here are in MB when unit says Mbyte
        out[k] = None if not rd else (sum(rd) + sum(wr)) / len(rd)
    traffic[cfg] = out

rep = G / "prof_c2_final.ncu-rep"
if rep.exists():
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rr[0], rr[1], rr[2:]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]
    idx = [hdr.index(w) for w in want if w in hdr]
    with open(P / "r01_ncu_c2_full.csv", "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow([hdr[i] for i in idx])
        w.writerow([units[i] for i in idx])
        c2 = {}
        for r in data:
            w.writerow([r[i] for i in idx])
            name = short(r[hdr.index("Kernel Name")])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(r[hdr.index("dram__bytes_read.sum")]) * scale[units[hdr.index("dram__bytes_read.sum")]]
            wr = float(r[hdr.index("dram__bytes_write.sum")]) * scale[units[hdr.index("dram__bytes_write.sum")]]
            c2[name] = rd + wr
        traffic["C2"] = c2

# the C3-C5 csv values: convert using their unit column
for cfg in ("C3", "C4", "C5"):
    f = G / f"traffic_{cfg}.csv"
    if not f.exists():
        continue
    acc = defaultdict(lambda: defaultdict(list))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    for r in rows(f):
        if r["Metric Name"].startswith("dram__bytes"):
            acc[short(r["Kernel Name"])][r["Metric Name"]].append(
                float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1))
    traffic[cfg] = {k: (sum(m["dram__bytes_read.sum"]) + sum(m["dram__bytes_write.sum"])) / len(m["dram__bytes_read.sum"])
                    for k, m in acc.items()}

traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes), from ncu "
                    "captures of tools/run_one.py (device-resident sort, one launch per kernel); "
                    "cold-cache, serialised")
(P / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1, sort_keys=True))
if (G / "launches_bench_c2.csv").exists():
    (P / "r01_launches_bench_c2.csv").write_text((G / "launches_bench_c2.csv").read_text())
print(json.dumps(traffic, indent=1))
