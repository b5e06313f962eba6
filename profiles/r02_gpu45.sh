# round 2, GPU call 45: broad phase staging the union of the warp's search boxes (cell table and
# particles) in shared memory, lanes scanning their own boxes from it: rebuild timing vs the
# per-thread broad phase, detection parity suites
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke45.log 2>&1; tail -1 gpurun_out/smoke45.log | cut -c1-100
timeout 600 python profiles/rebuild_timing.py --tag smem_broad > gpurun_out/rb45.log 2>&1
DEM_LIB_VARIANT=$V/libdem_ship.so timeout 600 python profiles/rebuild_timing.py --tag thread_broad >> gpurun_out/rb45.log 2>&1
grep '^{' gpurun_out/rb45.log; tail -2 gpurun_out/rb45.log
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_generator.py tests/test_gpu_bedbuilder.py -q -x -p no:cacheprovider > gpurun_out/broad_tests45.log 2>&1; tail -4 gpurun_out/broad_tests45.log
