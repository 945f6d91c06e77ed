#!/bin/bash
# ncu --set full of the TMA-in/STG-out fp32 quantile kernel and exp->normal, 1 GPU
mkdir -p gpurun_out/profiles
prof() {  # name regex kernel-arg [env]
  timeout 600 env $4 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 \
      -o gpurun_out/prof_$1 -f python tools/prof_kernel.py $3 3 > gpurun_out/profiles/ncu_$1.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_$1.ncu-rep > gpurun_out/profiles/ncu_$1.json 2>>gpurun_out/profiles/ncu_$1.log
}
prof tl_J k_normal_f32_tl stream_f32
prof tl_K k_normal_f32_tl stream_f32 QM_TL_CFG=K
prof exp2n_tl k_exp2n_f32_tl exp2n_f32
QM_TL_CFG=K timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_K.json 2>gpurun_out/bench_K.err
echo done
