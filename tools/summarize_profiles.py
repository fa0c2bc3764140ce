#!/usr/bin/env python
"""Turn ncu captures (gpurun_out/*.ncu-rep, launch-list CSVs) into the small tracked summaries under profiles/."""
import csv
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__warps_eligible.avg.per_cycle_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg", "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "smsp__sass_inst_executed_op_tmem_ldt.sum",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg",
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def summarize_rep(rep, dst, note):
    hdr, units, rows = raw_rows(rep)
    idx = {h: i for i, h in enumerate(hdr)}
    with open(dst, "w") as f:
        f.write(f"# {rep.name}\n{note}\n\n")
        for r in rows:
            f.write(f"kernel: {r[idx['Kernel Name']]}\n")
            for k in KEYS:
                if k in idx:
                    f.write(f"  {k:84s} {r[idx[k]]:>18s} {units[idx[k]]}\n")
            f.write("  warp stall samples (smsp__pcsamp_warps_issue_stalled_*):\n")
            stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), int(float(r[i]))) for h, i in idx.items()
                      if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued") and r[i]]
            tot = sum(v for _, v in stalls) or 1
            for name, v in sorted(stalls, key=lambda x: -x[1])[:9]:
                f.write(f"    {name:28s} {v:8d}  {100.0 * v / tot:5.1f} %\n")
            f.write("\n")


def summarize_launches(csv_path, dst, note):
    lines = [l for l in Path(csv_path).read_text().splitlines() if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] == "ns" else v
        name = r[ki].split("(")[0][:110]
        tot[name] += v
        cnt[name] += 1
    total = sum(tot.values())
    with open(dst, "w") as f:
        f.write(f"# {Path(csv_path).name}: kernel share of the profiled window\n{note}\n\n")
        f.write(f"{'kernel':112s} {'launches':>8s} {'total us':>12s} {'share':>7s}\n")
        for name, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"{name:112s} {cnt[name]:8d} {v:12.1f} {100 * v / total:6.2f}%\n")


if __name__ == "__main__":
    g = ROOT / "gpurun_out"
    p = ROOT / "profiles"
    p.mkdir(exist_ok=True)
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    names = {"c1": "C1, 16x{4,4} N=1e6 Q=1e3", "c2": "C2, 12x{6,5,5} N=1e7 Q=1e4 (default bench)",
             "c3": "C3, 8x{8,8} N=1e7 Q=1e4", "c4": "C4, 16x{4,4} N=2e8 Q=1e4", "c5": "C5, IVF K=16384 nprobe=64"}
    for rep in sorted(g.glob(f"{tag}_probe_*.ncu-rep")):
        summarize_rep(rep, p / (rep.stem + "_summary.txt"),
                      "ncu --set full --clock-control none --import-source on, the two probe_approx_umma_kernel launches "
                      "(class minima, candidate bitmaps) of `python bench.py --workload c5g --warmup 3`")
    for rep in sorted(g.glob(f"{tag}_scan_*.ncu-rep")):
        w = rep.stem.split("_")[-1]
        summarize_rep(rep, p / (rep.stem + "_summary.txt"),
                      f"ncu --set full --clock-control none --import-source on, one scan launch of "
                      f"`python bench.py --workload {w} --warmup 3` ({names.get(w, w)})")
    for lc in sorted(g.glob(f"{tag}_launches_*.csv")):
        w = lc.stem.split("_")[-1]
        (p / lc.name).write_text(lc.read_text())
        summarize_launches(lc, p / f"{tag}_launch_share_{w}.txt",
                           f"ncu --metrics gpu__time_duration.sum --clock-control none on `python bench.py --workload {w} "
                           f"--warmup 3 --no-cpu-baseline`, library kernels only (cold-cache, serialised per-launch times: "
                           f"compare SHARES, not absolutes)")
