for c in B H; do QM_TMA_CFG=$c python tools/exp_grid_ulp.py >> gpurun_out/exp.txt 2>&1; done
for c in H; do QM_TMA_CFG=$c timeout 300 python bench.py --no-variants --no-cpu-baseline > gpurun_out/ab_$c.json 2>gpurun_out/ab_$c.err; done
