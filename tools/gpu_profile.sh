# Round profile capture (one gpurun call per step: gpurun_out/ comes back only under 64 MiB).
#   bash tools/gpu_profile.sh bench    -> bench line + ncu launch list of the bench command
#   bash tools/gpu_profile.sh radix    -> ncu --set full of k_upfront + k_onesweep_t (radix, 1e8)
#   bash tools/gpu_profile.sh bucket   -> ncu --set full of k_bucket_segments (1e8)
set -x
case "$1" in
bench)
  python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1 ;;
radix)
  python tools/prof_sort.py --alg radix --reps 1 && \
  ncu --set full --import-source on --clock-control none -k regex:"k_onesweep_t|k_upfront" -c 2 \
      -o gpurun_out/r02_radix_${2:-cur} python tools/prof_sort.py --alg radix --reps 1 > gpurun_out/ncu_r.log 2>&1 ;;
bucket)
  python tools/prof_sort.py --alg bucket --reps 1 && \
  ncu --set full --import-source on --clock-control none -k regex:"k_bucket_segments" -c 1 \
      -o gpurun_out/r02_bucket_${2:-cur} python tools/prof_sort.py --alg bucket --reps 1 > gpurun_out/ncu_b.log 2>&1 ;;
esac
ls -la gpurun_out/
