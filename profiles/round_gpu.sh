# one GPU call: parity tests, the bench line, the sweep variants, launch list + full capture of the sweep
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
if [ "${NCU:-1}" = "1" ]; then
  python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/bench_profile.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/ncu_launch.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_sweep_t2 -s 500 -c 1 -o gpurun_out/prof_bench_sweep \
      python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/ncu_full.log 2>&1
fi
