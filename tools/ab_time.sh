#!/bin/bash
# Interleaved A/B of library builds on named hot-path calls (tools/time_variants.py):
#   NAMES="stream_f64 fused_f64" LIBS="paper_0901_0638_b200/ab/x.so" OUT=gpurun_out/ab bash tools/ab_time.sh
# The default build (libqm.so) runs first in every round; REPS rounds (default 3).
OUT=${OUT:-gpurun_out/ab}
mkdir -p $OUT
: > $OUT/ab_time.jsonl
for rep in $(seq ${REPS:-3}); do
  for lib in default ${LIBS}; do
    if [ $lib = default ]; then env=""; else env="QM_LIB_PATH=$lib"; fi
    env $env timeout 600 python tools/time_variants.py ${NAMES} 2>>$OUT/ab_time.err | \
      python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l); d['lib'] = '$lib'; d['rep'] = $rep; print(json.dumps(d))" >> $OUT/ab_time.jsonl
  done
done
python - "$OUT/ab_time.jsonl" <<'PY' > $OUT/ab_time_summary.txt
import json, sys, collections
rows = [json.loads(l) for l in open(sys.argv[1])]
g = collections.defaultdict(list)
for r in rows:
    g[(r['name'], r['lib'])].append(r['gsamples_s'])
for (n, lib), v in sorted(g.items()):
    print(f"{n:28s} {lib:50s} " + " ".join(f"{x:8.2f}" for x in v) + f"   median {sorted(v)[len(v)//2]:.2f}")
PY
cat $OUT/ab_time_summary.txt
