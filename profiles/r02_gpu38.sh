# round 2, GPU call 38: forward items with per-tile source lists, the wait and the forward-slot sums
# per warp after its items (no CTA-wide wait); diagnostic builds without the wait / without the
# forward sums (wrong results, timing bounds only) vs the shipped sweep
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke38.log 2>&1; tail -1 gpurun_out/smoke38.log
timeout 600 python profiles/sweep_ab.py --tag fwd_src > gpurun_out/ab38.log 2>&1
DEM_LIB_VARIANT=$V/libdem_nowait.so timeout 600 python profiles/sweep_ab.py --tag diag_nowait >> gpurun_out/ab38.log 2>&1
DEM_LIB_VARIANT=$V/libdem_nofsum.so timeout 600 python profiles/sweep_ab.py --tag diag_nofsum >> gpurun_out/ab38.log 2>&1
DEM_LIB_VARIANT=$V/libdem_ship.so timeout 600 python profiles/sweep_ab.py --tag ship >> gpurun_out/ab38.log 2>&1
grep '^{' gpurun_out/ab38.log; tail -3 gpurun_out/ab38.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_bench_column.py -q -x -p no:cacheprovider > gpurun_out/fwd_tests38.log 2>&1; tail -5 gpurun_out/fwd_tests38.log
