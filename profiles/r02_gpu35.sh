# round 2, GPU call 35: the sweep's plan invariants checked in-kernel (DEM_CHECK build, traps on violation) over
# the parity, decomposition, column and full-size tests, a ragged odd last tile, and the bench bed
set -x
mkdir -p gpurun_out
export DEM_LIB_VARIANT=paper_2501_05300_b200/lib/variants/libdem_check.so
timeout 300 python profiles/sanitize_run.py 1501 > gpurun_out/chk_small.log 2>&1; tail -2 gpurun_out/chk_small.log
timeout 300 python profiles/sweep_ab.py --tag check --n 20 > gpurun_out/chk_bench.log 2>&1; tail -2 gpurun_out/chk_bench.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_bench_column.py tests/test_gpu_gs.py tests/test_gpu_triaxial.py -q -x -p no:cacheprovider > gpurun_out/chk_tests.log 2>&1; tail -3 gpurun_out/chk_tests.log
