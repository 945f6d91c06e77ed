#!/bin/bash
# Interleaved A/B of QM_TL_CFG shapes on the headline bench (same box)
out=gpurun_out/ab_cfg.txt; : > $out
for rep in 1 2 3; do
  for c in ${CFGS:-L M N}; do
    QM_TL_CFG=$c timeout 300 python bench.py --no-variants --no-cpu-baseline --steps 100 > /tmp/ab.json 2>/tmp/ab.err
    python -c "
import json; d=json.loads(open('/tmp/ab.json').read().splitlines()[-1])
print('$rep', '$c', round(d['value'],1), round(d['roofline']['frac'],4))" >> $out 2>&1 || tail -3 /tmp/ab.err >> $out
  done
done
