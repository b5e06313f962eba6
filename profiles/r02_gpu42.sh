# round 2, GPU call 42: warp-cooperative smem-staged broad phase (north_star (b)): detection parity
# suites, rebuild timing vs the shipped per-thread broad phase, and the main-stage sweep ncu capture
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke42.log 2>&1; tail -1 gpurun_out/smoke42.log
timeout 600 python profiles/rebuild_timing.py --tag warp_broad > gpurun_out/rb42.log 2>&1
DEM_LIB_VARIANT=$V/libdem_ship.so timeout 600 python profiles/rebuild_timing.py --tag thread_broad >> gpurun_out/rb42.log 2>&1
grep '^{' gpurun_out/rb42.log; tail -2 gpurun_out/rb42.log
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_generator.py tests/test_gpu_bedbuilder.py tests/test_gpu_bench_column.py -q -x -p no:cacheprovider > gpurun_out/broad_tests42.log 2>&1; tail -4 gpurun_out/broad_tests42.log
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_sweep<\(bool\)0' --launch-skip 3 --launch-count 1 \
  -o gpurun_out/sweep_src42 -f python profiles/sweep_ab.py --n 3 --settle 10 > gpurun_out/ncu42.log 2>&1
tail -2 gpurun_out/ncu42.log
