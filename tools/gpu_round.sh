#!/bin/bash
# Round-end style session: GPU tests, smoke, full bench, reference arm, ncu of the
# changed kernels and the launch list of the headline bench.
mkdir -p gpurun_out/profiles
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench wall $(( $(date +%s) - t0 )) s" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
prof() {  # name regex [env] [prof_kernel name]
  timeout 600 env $3 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 \
      -o /tmp/prof_$1 -f python tools/prof_kernel.py ${4:-$1} 3 > gpurun_out/profiles/ncu_$1.log 2>&1
  python tools/ncu_summary.py /tmp/prof_$1.ncu-rep > gpurun_out/profiles/ncu_$1.json 2>>gpurun_out/profiles/ncu_$1.log
}
for k in ${PROFS:-}; do
  case $k in
    stream_f32) prof stream_f32 k_normal_f32_tl; cp /tmp/prof_stream_f32.ncu-rep gpurun_out/ ;;
    fused_f32) prof fused_f32 k_philox_f32 ;;
    mc) prof mc k_mc_call ;;
    config1_moro) prof config1_moro k_branchy ;;
    stream_f64) prof stream_f64 k_normal_f64_tl ;;
    fused_f64) prof fused_f64 k_philox_f64 ;;
    student) prof student k_student_f64_tl ;;
    exp2n_f32) prof exp2n_f32 k_exp2n_f32_tl ;;
    rode_hyp_f64) prof rode_hyp_f64 k_rode_map_tl ;;
    rode_philox_f32) prof rode_philox_f32 k_rode_philox ;;
    two_region) prof two_region k_normal_f32_tl "" stream_f32_two ;;
    student_moments) prof student_moments k_student_moments_tl ;;
  esac
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/profiles/ncu_bench.log 2>&1
cp /tmp/launches.csv gpurun_out/profiles/launches_bench.csv
python tools/ncu_summary.py --launches /tmp/launches.csv > gpurun_out/profiles/launches_bench_summary.json
echo done
