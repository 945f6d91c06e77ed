#!/bin/bash
# Interleaved A/B of library builds on the headline bench: LIBS="a.so b.so" (default lib = "default")
mkdir -p gpurun_out
out=gpurun_out/ab_libs.txt; : > $out
for rep in 1 2 3; do
  for lib in default ${LIBS}; do
    if [ $lib = default ]; then env=""; else env="QM_LIB_PATH=$lib"; fi
    env $env timeout 300 python bench.py --no-variants --no-cpu-baseline --steps 100 > /tmp/ab.json 2>/tmp/ab.err
    python -c "
import json; d=json.loads(open('/tmp/ab.json').read().splitlines()[-1])
print('$rep', '$lib', round(d['value'],1), round(d['roofline']['frac'],4))" >> $out 2>&1 || tail -3 /tmp/ab.err >> $out
  done
done
