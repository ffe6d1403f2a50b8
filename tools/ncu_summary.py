"""Summarise ncu evidence into profiles/ (run here, on the CPU box, on reports
brought back from a gpurun call):

  python tools/ncu_summary.py --rep gpurun_out/prof_blocked_r1.ncu-rep \
      --launches gpurun_out/launches_default.csv --tag r1 --key c5_fp64 --streams 8192

Writes profiles/<tag>_blocked_kernel.csv (raw metrics of interest),
profiles/<tag>_launches.md (per-kernel share of the bench command's launches) and
merges {key: {...}} into profiles/ncu_summary.json (read by bench.py)."""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "smsp__inst_executed.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = r[0], r[1], r[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def launches(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr, data = r, rows[i + 1:]
            break
    iK, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[r[iU]]
        k = r[iK].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += float(r[iV].replace(",", "")) * scale
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--key", required=True)
    ap.add_argument("--streams", type=int, required=True, help="streams in the profiled launch")
    ap.add_argument("--rows", type=int, default=1024)
    ap.add_argument("--alg-bytes-per-row", type=float, default=8 * (64 + 8), help="compulsory bytes per row")
    ap.add_argument("--job-streams", type=int, default=65536, help="streams of the benchmarked job")
    a = ap.parse_args()
    m = raw_metrics(a.rep)
    pdir = os.path.join(ROOT, "profiles")
    os.makedirs(pdir, exist_ok=True)
    with open(os.path.join(pdir, f"{a.tag}_blocked_kernel.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["metric", "unit", "value"])
        for k in KEYS:
            if k in m:
                w.writerow([k, m[k][1], m[k][0]])
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(m["dram__bytes_read.sum"][0]) * unit[m["dram__bytes_read.sum"][1]]
    wr = float(m["dram__bytes_write.sum"][0]) * unit[m["dram__bytes_write.sum"][1]]
    per_row = (rd + wr) / (a.streams * a.rows)
    summ_path = os.path.join(pdir, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    summ[a.key] = {
        "source": os.path.basename(a.rep), "profiled_streams": a.streams, "rows": a.rows,
        "dram_bytes_profiled_launch": rd + wr, "dram_bytes_per_row": per_row,
        "algorithmic_bytes_per_row": a.alg_bytes_per_row,
        "traffic_over_compulsory": per_row / a.alg_bytes_per_row,
        "note": f"dram_bytes_per_launch scales the per-row traffic of the profiled launch to {a.job_streams} streams",
        "dram_bytes_per_launch": per_row * a.job_streams * a.rows,
        "dmma_pipe_pct": m.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", ["?"])[0],
        "registers": m.get("launch__registers_per_thread", ["?"])[0],
        "warps_active_per_sm": m.get("sm__warps_active.avg.per_cycle_active", ["?"])[0],
    }
    json.dump(summ, open(summ_path, "w"), indent=1)
    if a.launches:
        agg = launches(a.launches)
        tot = sum(v[1] for v in agg.values())
        with open(os.path.join(pdir, f"{a.tag}_launches.md"), "w") as f:
            f.write(f"# ncu launch list ({os.path.basename(a.launches)}; cold-cache, serialised)\n\n")
            f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
            for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
                f.write(f"| `{k[:90]}` | {v[0]} | {v[1]:.3f} | {100 * v[1] / tot:.1f}% |\n")
    print(json.dumps(summ[a.key], indent=1))


if __name__ == "__main__":
    main()
