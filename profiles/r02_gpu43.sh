# round 2, GPU call 43: L2 prefetch of the next chunk's cross-tile partners (SWEEP_PF_L2=1) vs the
# shipped sweep (ncu: the first use of a gathered partner value holds 12 % of the stall samples);
# rebuild timing of the warp-cooperative broad phase vs the per-thread one
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 600 python profiles/sweep_ab.py --tag ship_warpbroad > gpurun_out/ab43.log 2>&1
DEM_LIB_VARIANT=$V/libdem_pfl2.so timeout 600 python profiles/sweep_ab.py --tag pf_l2 >> gpurun_out/ab43.log 2>&1
DEM_LIB_VARIANT=$V/libdem_ship.so timeout 600 python profiles/sweep_ab.py --tag ship >> gpurun_out/ab43.log 2>&1
DEM_LIB_VARIANT=$V/libdem_pfl2.so timeout 600 python profiles/sweep_ab.py --tag pf_l2_b >> gpurun_out/ab43.log 2>&1
grep '^{' gpurun_out/ab43.log; tail -2 gpurun_out/ab43.log
timeout 600 python profiles/rebuild_timing.py --tag warp_broad > gpurun_out/rb43.log 2>&1
DEM_LIB_VARIANT=$V/libdem_ship.so timeout 600 python profiles/rebuild_timing.py --tag thread_broad >> gpurun_out/rb43.log 2>&1
grep '^{' gpurun_out/rb43.log; tail -2 gpurun_out/rb43.log
