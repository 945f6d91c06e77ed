#!/bin/bash
# Round-2 session: GPU tests (all, no -x), smoke, diagnostics, full bench, reference
# arm, ncu --set full of every kernel family (pipe counters incl. FP64 instructions)
# and the launch list of the headline bench.   OUT=gpurun_out/<dir> PROFS=all|none
OUT=${OUT:-gpurun_out/r2}
mkdir -p $OUT/profiles
nvidia-smi -L > $OUT/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=20 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
for d in ${DIAG:-}; do timeout 300 python tools/student_diag.py $(echo $d | tr ',' ' ') >> $OUT/diag.txt 2>&1; done
if [ "${BENCH:-1}" = 1 ]; then
  t0=$(date +%s); timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench wall $(( $(date +%s) - t0 )) s" >> $OUT/bench.err
  timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
fi
prof() {  # name regex [env] [prof_kernel name]
  timeout 600 env $3 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 \
      -o /tmp/prof_$1 -f python tools/prof_kernel.py ${4:-$1} 3 > $OUT/profiles/ncu_$1.log 2>&1
  python tools/ncu_summary.py /tmp/prof_$1.ncu-rep > $OUT/profiles/ncu_$1.json 2>>$OUT/profiles/ncu_$1.log
}
want() { [ "${PROFS:-all}" = all ] || [[ " ${PROFS} " == *" $1 "* ]]; }
if [ "${PROFS:-all}" != all ] && [ "${PROFS}" != none ]; then
  want stream_f32 && { prof stream_f32 k_normal_f32_tl; cp /tmp/prof_stream_f32.ncu-rep $OUT/; }
  want stream_f64 && prof stream_f64 k_normal_f64_tl
  want fused_f64 && prof fused_f64 k_philox_f64
  want student && prof student k_student_f64_tl
  want student_moments && prof student_moments k_student_moments_tl
  want config1_breakless && prof config1_breakless "k_normal_f64" "" config1_breakless
  want fused_f32 && prof fused_f32 k_philox_f32
  want rode_hyp_f64 && prof rode_hyp_f64 k_rode_map_tl
  want student_rode && prof student_rode k_rode_map_tl
  want stream_f64_1212 && prof stream_f64_1212 k_normal_f64
  want rode_vg_real_f64 && prof rode_vg_real_f64 k_rode_map_tl
fi
if [ "${PROFS:-all}" = all ]; then
  prof stream_f32 k_normal_f32_tl; cp /tmp/prof_stream_f32.ncu-rep $OUT/
  prof stream_f64 k_normal_f64_tl
  prof stream_f64_1212 k_normal_f64
  prof fused_f32 k_philox_f32
  prof fused_f32_fma k_philox_f32 QM_LIB_PATH=paper_0901_0638_b200/ab/libqm_rat1.so fused_f32
  prof fused_f64 k_philox_f64
  prof student k_student_f64_tl
  prof student_k16 k_student_f64_tl
  prof student_rode k_rode_map_tl
  prof student_moments k_student_moments_tl
  prof moments k_moment_rows
  prof exp2n_f32 k_exp2n_f32_tl
  prof mc k_mc_call
  prof rode_hyp_f64 k_rode_map_tl
  prof rode_philox_f32 k_rode_philox
  prof two_region k_normal_f32_tl "" stream_f32_two
  for a in breakless as241 acklam refined moro breakless77; do
    prof config1_$a "k_normal_f64|k_branchy" "" config1_$a
    prof plain_config1_$a k_plain_f64 "" plain_config1_$a
  done
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-variants --no-cpu-baseline > $OUT/profiles/ncu_bench.log 2>&1
timeout 300 python tools/window_curve.py stream_f32 10,20,50,100,200,400,1000 > $OUT/window_curve.jsonl 2>&1
cp /tmp/launches.csv $OUT/profiles/launches_bench.csv
python tools/ncu_summary.py --launches /tmp/launches.csv > $OUT/profiles/launches_bench_summary.json
du -sh gpurun_out
echo done
