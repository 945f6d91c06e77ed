#!/bin/bash
# ncu --set full, one launch each, of every hot-path kernel family (1 GPU).
# Reports are summarised on the box (tools/ncu_summary.py); only the headline
# kernel's report is kept (gpurun_out/ is capped at 64 MiB).
mkdir -p gpurun_out/profiles
prof() {  # name regex [env] [prof_kernel name]
  timeout 600 env $3 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 \
      -o /tmp/prof_$1 -f python tools/prof_kernel.py ${4:-$1} 3 > gpurun_out/profiles/ncu_$1.log 2>&1
  python tools/ncu_summary.py /tmp/prof_$1.ncu-rep > gpurun_out/profiles/ncu_$1.json 2>>gpurun_out/profiles/ncu_$1.log
}
prof stream_f32 k_normal_f32_tl
cp /tmp/prof_stream_f32.ncu-rep gpurun_out/ 2>/dev/null
prof stream_f32_tma k_normal_f32_tma QM_STREAM_PATH=tma stream_f32
prof stream_f32_ldg k_normal_f32 QM_STREAM_PATH=ldg stream_f32
prof stream_f64 k_normal_f64_tl
prof fused_f32 k_philox_f32
prof fused_f64 k_philox_f64
prof student k_student_f64
prof exp2n_f32 k_exp2n_f32_tl
prof moments k_moment_rows
prof mc k_mc_call
prof config1_breakless k_normal_f64
prof config1_as241 k_branchy
prof config1_acklam k_branchy
prof config1_refined k_branchy
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/profiles/ncu_bench.log 2>&1
cp /tmp/launches.csv gpurun_out/profiles/launches_bench.csv
python tools/ncu_summary.py --launches /tmp/launches.csv > gpurun_out/profiles/launches_bench_summary.json
du -sh gpurun_out
echo done
