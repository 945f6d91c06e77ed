"""Summarise ncu reports / launch lists into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py report.ncu-rep [...]     -> one JSON object per kernel
    python tools/ncu_summary.py --launches launches.csv   -> per-kernel share of device time
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_of_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "divergent_branch_targets": "smsp__sass_branch_targets_threads_divergent.sum",
    "threads_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "warp_inst_executed": "smsp__inst_executed.sum",
    "fp64_inst_executed": "smsp__inst_executed_pipe_fp64.sum",
    "fma_cycles_active": "sm__pipe_fma_cycles_active.sum",
    "sm_clock_hz": "sm__cycles_elapsed.avg.per_second",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smem_pipe_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
UNIT_SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "us": 1.0, "ms": 1e3, "ns": 1e-3,
              "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "?"), "report": rep.split("/")[-1]}
        for name, key in KEYS.items():
            if key in d and d[key] not in ("", "n/a"):
                try:
                    v = float(d[key].replace(",", ""))
                except ValueError:
                    continue
                k[name] = v * UNIT_SCALE.get(u.get(key, ""), 1.0)
        stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v)
                  for h, v in d.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not h.endswith("not_issued") and v.replace(".", "", 1).isdigit()}
        tot = sum(stalls.values()) or 1.0
        k["stall_pct_top"] = {s: round(100 * v / tot, 1) for s, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]}
        res.append(k)
    return res


def launches(path):
    per = defaultdict(lambda: [0, 0.0])
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        per[name][0] += 1
        per[name][1] += float(r["Metric Value"].replace(",", "")) * (1e-3 if r.get("Metric Unit") == "ns" else 1.0)
    tot = sum(v[1] for v in per.values())
    return {k: {"launches": v[0], "total_us": round(v[1], 1), "share": round(v[1] / tot, 4)}
            for k, v in sorted(per.items(), key=lambda x: -x[1][1])}


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        allk = []
        for rep in sys.argv[1:]:
            allk += summarise(rep)
        print(json.dumps(allk, indent=1))
