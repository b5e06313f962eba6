# round 2, first GPU call: GPU tests (no -x: full picture), bench line, launch list, sweep capture
set -x
mkdir -p gpurun_out
export DEM_DEBUG=
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -30 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
DEM_DEBUG=1 timeout 300 python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/bench_profile.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 300 -c 1 -o gpurun_out/prof_sweep_r02a \
    python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
