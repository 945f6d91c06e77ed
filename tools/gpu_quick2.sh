#!/bin/bash
# Quick GPU iteration: selected pytest files, a short variant timing, optional ncu captures.
#   OUT=gpurun_out/<dir> TESTS="tests/a.py tests/b.py" VARS=1 PROFS="name:regex ..."
OUT=${OUT:-gpurun_out/q}
mkdir -p $OUT/profiles
if [ -n "${TESTS:-}" ]; then
  timeout 1500 python -m pytest $TESTS -m gpu -q -rf -x > $OUT/pytest.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest.txt
fi
if [ -n "${TIME:-}" ]; then timeout 900 python tools/time_variants.py $TIME > $OUT/time.json 2> $OUT/time.err; fi
for pr in ${PROFS:-}; do
  name=${pr%%:*}; rx=${pr#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s 1 -c 1 \
      -o $OUT/prof_$name -f python tools/prof_kernel.py $name 3 > $OUT/profiles/ncu_$name.log 2>&1
  python tools/ncu_summary.py $OUT/prof_$name.ncu-rep > $OUT/profiles/ncu_$name.json 2>>$OUT/profiles/ncu_$name.log
done
echo done
