#!/bin/bash
# ncu --set full, one launch each, of every hot-path kernel family (1 GPU).
mkdir -p gpurun_out
prof() {  # name regex
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 \
      -o gpurun_out/prof_$1 -f python tools/prof_kernel.py $1 3 > gpurun_out/ncu_$1.log 2>&1
}
prof stream_f32 k_normal_f32_tma
QM_STREAM_PATH=ldg timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_normal_f32 -s 1 -c 1 \
    -o gpurun_out/prof_stream_f32_ldg -f python tools/prof_kernel.py stream_f32 3 > gpurun_out/ncu_ldg.log 2>&1
prof stream_f64 k_normal_f64
prof fused_f32 k_philox_f32
prof fused_f64 k_philox_f64
prof student k_student_f64
prof exp2n_f32 k_exp2n_f32_tma
prof moments k_moment_rows
prof mc k_mc_call
prof config1_breakless k_normal_f64
prof config1_as241 k_branchy
prof config1_acklam k_branchy
prof config1_refined k_branchy
echo done
