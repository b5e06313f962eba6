# round 2, GPU call 50: warp ranges of a tile balanced by a per-item cost (intra / cross / boundary
# weights) instead of the item count (ncu: 8 % of the stall samples at the tile barrier) vs shipped
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 600 python profiles/sweep_ab.py --tag ship > gpurun_out/ab50.log 2>&1
for t in ws463 ws483 ws452; do DEM_LIB_VARIANT=$V/libdem_$t.so timeout 600 python profiles/sweep_ab.py --tag $t >> gpurun_out/ab50.log 2>&1; done
timeout 600 python profiles/sweep_ab.py --tag ship_b >> gpurun_out/ab50.log 2>&1
DEM_LIB_VARIANT=$V/libdem_ws463.so timeout 600 python profiles/sweep_ab.py --tag ws463_b >> gpurun_out/ab50.log 2>&1
grep '^{' gpurun_out/ab50.log; tail -2 gpurun_out/ab50.log
