# round 2, GPU call 39: forward items with 64-byte forward slots (full-sector stores), forward-first
# warp order (default) and natural owner order (SWEEP_NOSPLIT) vs the shipped sweep
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke39.log 2>&1; tail -1 gpurun_out/smoke39.log
timeout 600 python profiles/sweep_ab.py --tag fwd64 > gpurun_out/ab39.log 2>&1
DEM_LIB_VARIANT=$V/libdem_nosplit.so timeout 600 python profiles/sweep_ab.py --tag fwd64_nosplit >> gpurun_out/ab39.log 2>&1
DEM_LIB_VARIANT=$V/libdem_ship.so timeout 600 python profiles/sweep_ab.py --tag ship >> gpurun_out/ab39.log 2>&1
grep '^{' gpurun_out/ab39.log; tail -3 gpurun_out/ab39.log
