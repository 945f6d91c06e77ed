#!/bin/bash
# (build the A/B libraries first: python -c "from paper_0901_0638_b200 import build as b; b.build(out='build/libqm_kc9.so', defines=['QM_D13_KC=9'])", likewise kc8)
# fp64 D13: compensated-step count A/B (parity + speed)
for lib in default build/libqm_kc9.so build/libqm_kc8.so; do
  if [ $lib = default ]; then env=""; else env="QM_LIB_PATH=$lib"; fi
  env $env timeout 600 python -m pytest tests/test_gpu_normal.py -q -k "float64 or fp64" -rf > gpurun_out/pytest_kc_$(basename $lib).txt 2>&1
  env $env timeout 120 python tools/time_op.py stream_f64 10 >> gpurun_out/t_kc.txt 2>&1
  env $env timeout 120 python tools/time_op.py fused_f64 5 >> gpurun_out/t_kc.txt 2>&1
done
