# round 2, GPU call 48: item records and impulses with an L2 evict-first policy (SWEEP_L2HINT=1), so the
# 8.9 GB per sweep of streaming records do not displace the particle states the cross-tile partner
# gathers re-read (L2 hit rate 21 %), vs the shipped sweep; ncu L2 hit rate of both
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
DEM_LIB_VARIANT=$V/libdem_l2hint.so timeout 600 python profiles/sweep_ab.py --tag l2hint > gpurun_out/ab48.log 2>&1
timeout 600 python profiles/sweep_ab.py --tag ship >> gpurun_out/ab48.log 2>&1
DEM_LIB_VARIANT=$V/libdem_l2hint.so timeout 600 python profiles/sweep_ab.py --tag l2hint_b >> gpurun_out/ab48.log 2>&1
timeout 600 python profiles/sweep_ab.py --tag ship_b >> gpurun_out/ab48.log 2>&1
grep '^{' gpurun_out/ab48.log; tail -2 gpurun_out/ab48.log
for L in ship:paper_2501_05300_b200/lib/libdem.so l2hint:$V/libdem_l2hint.so; do
  tag=${L%%:*}; lib=${L#*:}
  DEM_LIB_VARIANT=$lib timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base demangled -k 'regex:k_sweep<\(bool\)0' --launch-skip 3 --launch-count 2 --csv --log-file gpurun_out/l2_48_$tag.csv python profiles/sweep_ab.py --n 3 --settle 10 > /dev/null 2>&1
done
