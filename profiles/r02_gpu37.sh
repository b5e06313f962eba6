# round 2, GPU call 37: every contact evaluated once per sweep (forward items, the partner's share
# delivered through a global forward slot, lower tiles' forward phases awaited before the final
# phase) vs the shipped contact-once-per-tile sweep: smoke, A/B timing, parity suites
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke37.log 2>&1; tail -3 gpurun_out/smoke37.log
timeout 600 python profiles/sweep_ab.py --tag fwd > gpurun_out/ab37.log 2>&1
DEM_LIB_VARIANT=$V/libdem_ship.so timeout 600 python profiles/sweep_ab.py --tag ship >> gpurun_out/ab37.log 2>&1
timeout 600 python profiles/sweep_ab.py --tag fwd2 >> gpurun_out/ab37.log 2>&1
grep '^{' gpurun_out/ab37.log; tail -5 gpurun_out/ab37.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_bench_column.py tests/test_gpu_gs.py tests/test_gpu_protocol.py -q -x -p no:cacheprovider > gpurun_out/fwd_tests.log 2>&1; tail -15 gpurun_out/fwd_tests.log
