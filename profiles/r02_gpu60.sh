# round 2, GPU call 60: two sweep CTAs in the 132 KB configuration without losing slots:
# int16 scale exponents + bad-flag bitmask (SWEEP_SIG16=1, -4 KB per CTA) with slot capacity
# 664 / 680 (g664, g680) and 768 (g768: the code change alone, 164 KB configuration)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
export DEM_DEBUG=1
for tag in ship g664 g680 g768 ship_b g664_b g680_b g768_b; do
  case $tag in ship*) unset DEM_LIB_VARIANT;; g664*) export DEM_LIB_VARIANT=$V/libdem_g664.so;; g680*) export DEM_LIB_VARIANT=$V/libdem_g680.so;; g768*) export DEM_LIB_VARIANT=$V/libdem_g768.so;; esac
  timeout 600 python profiles/sweep_ab.py --tag $tag >> gpurun_out/ab60.log 2>&1
done
for tag in c3ship c3g664 c3g680; do
  case $tag in c3ship) unset DEM_LIB_VARIANT;; c3g664) export DEM_LIB_VARIANT=$V/libdem_g664.so;; c3g680) export DEM_LIB_VARIANT=$V/libdem_g680.so;; esac
  timeout 600 python profiles/sweep_ab.py --workload config3-geom --tag $tag >> gpurun_out/ab60.log 2>&1
done
unset DEM_LIB_VARIANT DEM_DEBUG
grep -E '^\{|dem_bench' gpurun_out/ab60.log | cut -c1-160
DEM_LIB_VARIANT=$V/libdem_g680.so timeout 900 ncu --metrics launch__shared_mem_config_size,launch__occupancy_limit_shared_mem,l1tex__t_sector_hit_rate.pct,gpu__time_duration.sum \
    --clock-control none -k regex:k_sweep -s 1200 -c 1 --csv python profiles/sweep_ab.py --tag ncu_g680 --n 10 > gpurun_out/ncu60_g680.csv 2> gpurun_out/ncu60_g680.err
grep -E "config_size|limit_shared|hit_rate|duration" gpurun_out/ncu60_g680.csv | awk -F'","' '{print $(NF-3), $NF}'
DEM_LIB_VARIANT=$V/libdem_g664.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_bench_column.py -q -x -p no:cacheprovider > gpurun_out/g664_tests60.log 2>&1; tail -3 gpurun_out/g664_tests60.log
