# round 2, GPU call 59: a smaller shared-memory footprint per sweep CTA so that two CTAs fit the
# 132 KB carveout (L1 92 -> 124 KB; GPU call 58: the 228 KB carveout, L1 28 KB, is 11 % slower):
# the bad-share flags as a bitmask (shipped candidate) and the slot capacity 600 / 576 (variants)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
export DEM_DEBUG=1
for tag in ship s600 s576 ship_b s600_b s576_b; do
  case $tag in ship*) unset DEM_LIB_VARIANT;; s600*) export DEM_LIB_VARIANT=$V/libdem_s600.so;; s576*) export DEM_LIB_VARIANT=$V/libdem_s576.so;; esac
  timeout 600 python profiles/sweep_ab.py --tag $tag >> gpurun_out/ab59.log 2>&1
done
for tag in c3ship c3s576; do
  case $tag in c3ship) unset DEM_LIB_VARIANT;; c3s576) export DEM_LIB_VARIANT=$V/libdem_s576.so;; esac
  timeout 600 python profiles/sweep_ab.py --workload config3-geom --tag $tag >> gpurun_out/ab59.log 2>&1
done
unset DEM_LIB_VARIANT DEM_DEBUG
grep -E '^\{|items' gpurun_out/ab59.log | cut -c1-160
for v in s600 s576; do
  DEM_LIB_VARIANT=$V/libdem_$v.so timeout 900 ncu --metrics launch__shared_mem_config_size,launch__occupancy_limit_shared_mem,l1tex__t_sector_hit_rate.pct,gpu__time_duration.sum \
    --clock-control none -k regex:k_sweep -s 1200 -c 1 --csv python profiles/sweep_ab.py --tag ncu_$v --n 10 > gpurun_out/ncu59_$v.csv 2> gpurun_out/ncu59_$v.err
  grep -E "config_size|limit_shared|hit_rate|duration" gpurun_out/ncu59_$v.csv | awk -F'","' '{print $(NF-2), $NF}'
done
DEM_LIB_VARIANT=$V/libdem_s600.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/s600_tests59.log 2>&1; tail -3 gpurun_out/s600_tests59.log
