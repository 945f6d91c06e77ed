#!/bin/bash
# A/B the fp32 streaming pipeline shapes (QM_TMA_CFG) and the LDG path.
mkdir -p gpurun_out
for cfg in A B C; do
  QM_TMA_CFG=$cfg timeout 300 python bench.py --no-variants --no-cpu-baseline > gpurun_out/ab_$cfg.json 2>gpurun_out/ab_$cfg.err
done
QM_STREAM_PATH=ldg timeout 300 python bench.py --no-variants --no-cpu-baseline > gpurun_out/ab_ldg.json 2>gpurun_out/ab_ldg.err
for cfg in B C; do
QM_TMA_CFG=$cfg timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_normal_f32_tma -s 1 -c 1 \
    -o gpurun_out/prof_tma_$cfg -f python tools/prof_kernel.py stream_f32 3 > gpurun_out/ncu_$cfg.log 2>&1
done
QM_STREAM_PATH=ldg timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_normal_f32 -s 1 -c 1 \
    -o gpurun_out/prof_ldg -f python tools/prof_kernel.py stream_f32 3 > gpurun_out/ncu_ldg.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
