#!/bin/bash
# A/B the fp32 streaming pipelines and (optionally) an experimental library build.
mkdir -p gpurun_out
rm -f gpurun_out/ab_*.json
timeout 600 python -m pytest tests/test_gpu_normal.py tests/test_gpu_tail.py -q -rf > gpurun_out/pytest_ab.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.txt
for cfg in ${CFGS:-J K L}; do
  QM_TL_CFG=$cfg timeout 300 python bench.py --no-variants --no-cpu-baseline > gpurun_out/ab_$cfg.json 2>gpurun_out/ab_$cfg.err
done
for lib in ${LIBS:-}; do
  n=$(basename $lib .so)
  QM_LIB_PATH=$lib timeout 600 python -m pytest tests/test_gpu_normal.py -q -rf > gpurun_out/pytest_$n.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_$n.txt
  QM_LIB_PATH=$lib timeout 300 python tools/exp_grid_ulp.py > gpurun_out/grid_$n.txt 2>&1
  for cfg in ${LCFGS:-J L M}; do
    QM_LIB_PATH=$lib QM_TL_CFG=$cfg timeout 300 python bench.py --no-variants --no-cpu-baseline > gpurun_out/ab_${n}_$cfg.json 2>gpurun_out/ab_${n}_$cfg.err
  done
done
python - <<'PY' > gpurun_out/ab_summary.txt
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*.json")):
    try:
        d = json.loads(open(f).read().splitlines()[-1])
        print(f, round(d["value"], 1), round(d["roofline"]["frac"], 4))
    except Exception as e:
        print(f, "ERR", e)
PY
