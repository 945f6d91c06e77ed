#!/bin/bash
# One GPU session: tests, bench, launch list and one ncu --set full capture.
# usage: tools/gpu_check.sh [kernel-regex] [prof_kernel.py name]
set -x
KRE=${1:-k_normal_f32_tma}
KNAME=${2:-stream_f32}
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
for cfg in A B E; do
  QM_TMA_CFG=$cfg timeout 300 python bench.py --no-variants --no-cpu-baseline > gpurun_out/ab_$cfg.json 2>gpurun_out/ab_$cfg.err
done
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 1 --no-variants --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 1 -c 1 \
    -o gpurun_out/prof_$KNAME -f python tools/prof_kernel.py $KNAME 3 > gpurun_out/ncu_full.log 2>&1
echo done
