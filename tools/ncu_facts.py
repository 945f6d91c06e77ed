"""profiles/<round>/ncu_*.json -> profiles/ncu_traffic.json: per-sample DRAM bytes and
warp-instructions of each hot-path kernel (bench.py reads it for `roofline.traffic`
and the issue-slot rooflines of the compute-bound rows).

    python tools/ncu_facts.py profiles/r01
"""
import json
import os
import sys

# elements per captured launch (tools/prof_kernel.py)
ELEMS = {"stream_f32": 1 << 28, "stream_f32_ldg": 1 << 28, "stream_f64": 1 << 28, "fused_f32": 1 << 32,
         "fused_f64": 1 << 31, "student": 1 << 30, "exp2n_f32": 1 << 28, "moments": 1 << 30, "mc": 1 << 32,
         "student_moments": 1 << 30, "two_region": 1 << 28, "rode_hyp_f64": 1 << 28, "rode_philox_f32": 1 << 28,
         "stream_f64_1212": 1 << 28, "fused_f32_fma": 1 << 32, "student_k16": 1 << 30, "student_rode": 1 << 30,
         "rode_vg_real_f64": 1 << 28}
for _a in ("breakless", "as241", "acklam", "refined", "moro", "breakless77"):      # config 1: one launch of 2^20
    ELEMS[f"config1_{_a}"] = 1 << 20
    ELEMS[f"plain_config1_{_a}"] = 1 << 20

d = sys.argv[1]
out = {}
for name, n in ELEMS.items():
    p = os.path.join(d, f"ncu_{name}.json")
    if not os.path.exists(p):
        continue
    k = json.load(open(p))[0]
    out[name] = {"kernel": k["kernel"],
                 "dram_bytes_per_elem": (k.get("dram_read_bytes", 0) + k.get("dram_write_bytes", 0)) / n,
                 "warp_inst_per_elem": k.get("warp_inst_executed", 0) / n,
                 # FP64-pipe warp-instructions per sample: the pipe's % of its peak
                 # (0.5 warp-inst/cycle/SMSP, 592 SMSPs) x the launch's cycles (ncu duration x clock)
                 "fp64_inst_per_elem": (k.get("fp64_pipe_pct", 0) / 100 * 592 * 0.5 *
                                        k.get("duration_us", 0) * 1e-6 * k.get("sm_clock_hz", 0) / n),
                 "source": f"{p} (ncu --set full, one launch of {n} samples)"}
    if k.get("smem_wavefronts"):       # shared-memory data-pipe wavefronts (the RODE maps' gathers)
        out[name]["smem_wavefronts_per_elem"] = k["smem_wavefronts"] / n
    for key in ("fp64_pipe_pct", "fma_pipe_pct", "alu_pipe_pct", "xu_pipe_pct", "issue_active_pct",
                "divergent_branch_targets", "threads_per_inst", "registers", "smem_pipe_pct"):
        if key in k:
            out[name][key] = k[key]
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
