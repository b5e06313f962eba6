# round 2, GPU call 56: persistent CTAs with dynamic tiles (global counter reset by the last CTA), the
# next tile staged by TMA into the second buffer, and each warp requesting the next tile's warp range
# and first records before the tile's final barrier (SWEEP_PERSIST=1) vs the shipped sweep; parity
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
DEM_LIB_VARIANT=$V/libdem_pdyn.so timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke56.log 2>&1; tail -1 gpurun_out/smoke56.log | cut -c1-150
timeout 600 python profiles/sweep_ab.py --tag ship > gpurun_out/ab56.log 2>&1
DEM_LIB_VARIANT=$V/libdem_pdyn.so timeout 600 python profiles/sweep_ab.py --tag pers_dyn >> gpurun_out/ab56.log 2>&1
timeout 600 python profiles/sweep_ab.py --tag ship_b >> gpurun_out/ab56.log 2>&1
DEM_LIB_VARIANT=$V/libdem_pdyn.so timeout 600 python profiles/sweep_ab.py --tag pers_dyn_b >> gpurun_out/ab56.log 2>&1
grep '^{' gpurun_out/ab56.log; tail -2 gpurun_out/ab56.log
DEM_LIB_VARIANT=$V/libdem_pdyn.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_bench_column.py -q -x -p no:cacheprovider > gpurun_out/pdyn_tests56.log 2>&1; tail -3 gpurun_out/pdyn_tests56.log
