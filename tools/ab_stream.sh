#!/bin/bash
# A/B the fp32 streaming pipeline shapes (QM_TMA_CFG) + tests + full bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
for cfg in ${CFGS:-B F G}; do
  QM_TMA_CFG=$cfg timeout 300 python bench.py --no-variants --no-cpu-baseline > gpurun_out/ab_$cfg.json 2>gpurun_out/ab_$cfg.err
done
