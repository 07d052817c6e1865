"""Round-2 summaries: turns the gpurun_out/r02_* captures (tools/gpu_profile_r02.sh)
into committed files under profiles/:
  profiles/ncu_traffic.json           DRAM bytes (read + write) per launch, per config and kernel (C1-C5)
  profiles/r02_ncu_c2_full.csv        key metrics of the C2 ncu --set full captures (KB3, KB4, fused KF)
  profiles/r02_ncu_*_lines.txt        per-source-line stall / instruction / SMEM-wavefront shares
  profiles/r02_launches_bench_c2.csv  the launch list of `python bench.py` (C2)
"""
import csv
import io
import json
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
G = ROOT / "gpurun_out"
P = ROOT / "profiles"

SHORT = {"bucket_partition": "bucket_partition", "bucket_sort": "bucket_sort", "bucket_hist": "bucket_hist",
         "bucket_colscan": "bucket_colscan", "scatter_kernel": "bitset_scatter", "scan2_kernel": "bitset_scan",
         "scan_kernel": "bitset_scan", "fused_sort": "fused_sort", "key_max": "key_max",
         "small_sort": "small_sort"}


def short(name: str) -> str:
    for k, v in SHORT.items():
        if k in name:
            return v
    return name[:40]


def csv_rows(path: Path):
    lines = [l for l in path.read_text().splitlines() if l.startswith('"')]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


def traffic():
    out = json.loads((P / "ncu_traffic.json").read_text()) if (P / "ncu_traffic.json").exists() else {}
    for cfg in ("C1", "C2", "C3", "C4", "C5"):
        f = G / f"r02_traffic_{cfg}.csv"
        if not f.exists():
            continue
        acc = defaultdict(lambda: defaultdict(list))
        for r in csv_rows(f):
            acc[short(r["Kernel Name"])][r["Metric Name"]].append(float(r["Metric Value"].replace(",", "")))
        per = {}
        for k, m in acc.items():
            rd, wr = m.get("dram__bytes_read.sum", []), m.get("dram__bytes_write.sum", [])
            if rd:
                per[k] = (sum(rd) + sum(wr)) / len(rd)
        out[cfg] = per
    (P / "ncu_traffic.json").write_text(json.dumps(out, indent=1) + "\n")


WANT = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]


def full_metrics():
    rows = []
    for rep in ("r02_prof_c2.ncu-rep", "r02_prof_kf_c2.ncu-rep", "r02_prof_ks_c1.ncu-rep"):
        f = G / rep
        if not f.exists():
            continue
        t = subprocess.run(["ncu", "-i", str(f), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(io.StringIO(t)))
        hdr, units, data = rr[0], rr[1], rr[2:]
        for d in data:
            rows.append({w: (d[hdr.index(w)] + (" " + units[hdr.index(w)] if units[hdr.index(w)] else ""))
                         for w in WANT if w in hdr} | {"capture": rep})
    if rows:
        with open(P / "r02_ncu_c2_full.csv", "w", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=["capture"] + WANT)
            w.writeheader()
            w.writerows(rows)


def lines():
    tool = ROOT / "tools" / "ncu_lines.py"
    for rep, kern, name in (("r02_prof_c2.ncu-rep", "bucket_partition", "r02_ncu_c2_kb3_lines.txt"),
                            ("r02_prof_c2.ncu-rep", "bucket_sort", "r02_ncu_c2_kb4_lines.txt"),
                            ("r02_prof_kf_c2.ncu-rep", "fused", "r02_ncu_kf_c2_lines.txt"),
                            ("r02_prof_ks_c1.ncu-rep", "small_sort", "r02_ncu_ks_c1_lines.txt")):
        if (G / rep).exists():
            t = subprocess.run([sys.executable, str(tool), str(G / rep), kern, "30"], capture_output=True,
                               text=True).stdout
            (P / name).write_text(t)


def stalls():
    """Warp-stall reasons per issued instruction and pipe utilisation of the C2 kernels and KS."""
    keys = ["smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    out = []
    for rep in ("r02_prof_c2.ncu-rep", "r02_prof_ks_c1.ncu-rep"):
        f = G / rep
        if not f.exists():
            continue
        t = subprocess.run(["ncu", "-i", str(f), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(io.StringIO(t)))
        hdr, data = rr[0], rr[2:]
        for d in data:
            row = dict(zip(hdr, d))
            out.append(f"== {row['Kernel Name'][:70]}  {row.get('gpu__time_duration.sum')} us")
            st = []
            for k, v in row.items():
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") \
                        and "not_issued" not in k:
                    try:
                        st.append((float(v.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            for v, k in sorted(st, reverse=True)[:9]:
                out.append(f"   {v:7.3f} warps stalled per issued instruction: {k}")
            for k in keys:
                if k in row:
                    out.append(f"   {row[k]:>10s}  {k}")
    if out:
        (P / "r02_ncu_stalls.txt").write_text("\n".join(out) + "\n")


if __name__ == "__main__":
    traffic()
    full_metrics()
    lines()
    stalls()
    for src, dst in (("r02_launches_bench_c2.csv", "r02_launches_bench_c2.csv"),
                     ("r02_bench_c2.json", "r02_bench_c2.json"), ("r02_bench_all.jsonl", "r02_bench_all.jsonl"),
                     ("r02_bench_reference.json", "r02_bench_reference_arm.json"),
                     ("r02_bench_c1_ks.json", "r02_bench_c1_ks.json"),
                     ("r02_bench_c4_chunked.json", "r02_bench_c4_chunked.json"),
                     ("r02_bench_c5_chunked.json", "r02_bench_c5_chunked.json"),
                     ("r02_width_bench.jsonl", "r02_width_bench.jsonl")):
        if (G / src).exists():
            shutil.copy(G / src, P / dst)
    print("ok")
