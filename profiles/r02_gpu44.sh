# round 2, GPU call 44: rebuild-phase timing, warp-cooperative smem-staged broad phase vs the
# per-thread one (profiles/rebuild_timing.py on config4-geom)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 600 python profiles/rebuild_timing.py --tag warp_broad > gpurun_out/rb44.log 2>&1
DEM_LIB_VARIANT=$V/libdem_ship.so timeout 600 python profiles/rebuild_timing.py --tag thread_broad >> gpurun_out/rb44.log 2>&1
timeout 600 python profiles/rebuild_timing.py --tag warp_broad_b >> gpurun_out/rb44.log 2>&1
grep '^{' gpurun_out/rb44.log; tail -2 gpurun_out/rb44.log
