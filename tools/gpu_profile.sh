set -x
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -c 3000 gpurun_out/bench_default.json
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
python tools/prof_sort.py --alg radix --reps 1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_onesweep|k_upfront" -c 2 -o gpurun_out/r02_radix python tools/prof_sort.py --alg radix --reps 1 > gpurun_out/ncu_r.log 2>&1
python tools/prof_sort.py --alg bucket --reps 1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_bucket_segments" -c 1 -o gpurun_out/r02_bucket python tools/prof_sort.py --alg bucket --reps 1 > gpurun_out/ncu_b.log 2>&1
ls -la gpurun_out/
