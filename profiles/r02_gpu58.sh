# round 2, GPU call 58: the sweep's shared-memory carveout (DEM_SWEEP_CARVEOUT, percent of the unified
# L1/shared capacity; 2 CTAs need ~150 KB) against the driver's default choice: A/B with
# profiles/sweep_ab.py, and the configured size and L1 hit rate from ncu
set -x
mkdir -p gpurun_out
for tag in ship cv66 cv100 ship_b cv66_b cv72; do
  case $tag in ship*) unset DEM_SWEEP_CARVEOUT;; cv66*) export DEM_SWEEP_CARVEOUT=66;; cv100) export DEM_SWEEP_CARVEOUT=100;; cv72) export DEM_SWEEP_CARVEOUT=72;; esac
  timeout 600 python profiles/sweep_ab.py --tag $tag >> gpurun_out/ab58.log 2>&1
done
unset DEM_SWEEP_CARVEOUT
grep '^{' gpurun_out/ab58.log | cut -c1-200; tail -2 gpurun_out/ab58.log
for cv in default 66 100; do
  if [ $cv = default ]; then unset DEM_SWEEP_CARVEOUT; else export DEM_SWEEP_CARVEOUT=$cv; fi
  timeout 900 ncu --metrics launch__shared_mem_config_size,launch__occupancy_limit_shared_mem,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,dram__bytes_read.sum \
    --clock-control none -k regex:k_sweep -s 1200 -c 1 --csv python profiles/sweep_ab.py --tag ncu_$cv --n 10 > gpurun_out/ncu58_$cv.csv 2> gpurun_out/ncu58_$cv.err
  grep -E "config_size|limit_shared|warps_active|hit_rate|duration|dram" gpurun_out/ncu58_$cv.csv | awk -F'","' '{print $(NF-2), $NF}' | cut -c1-120
done
