# round 2: the evidence call -- GPU tests, bench lines (default workload with plates, config4-count),
# the launch list and a full ncu capture of the sweep inside the bench
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_curves_mini.py > gpurun_out/gpu_tests_round.log 2>&1; tail -5 gpurun_out/gpu_tests_round.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_round.json 2> gpurun_out/bench_round.err; cat gpurun_out/bench_round.json; tail -3 gpurun_out/bench_round.err
timeout 1500 python bench.py --workload config4-count --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_count.json 2> gpurun_out/bench_count.err; cat gpurun_out/bench_count.json; tail -3 gpurun_out/bench_count.err
timeout 600 python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/bench_profile.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_round.csv \
    python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/ncu_launch.log 2>&1
timeout 600 python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/bench_profile2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 600 -c 1 -o gpurun_out/prof_bench_sweep_r02 \
    python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
