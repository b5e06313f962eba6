# round 2, GPU call 46: broad-phase kernel times (ncu launch list, k_broad only) of the per-thread
# scan (shipped round-2 library), the smem-staged warp scan (320-particle boxes, 128 registers) and
# the same at 192 particles and 6 CTAs per SM
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
for L in ship:$V/libdem_ship.so smem:paper_2501_05300_b200/lib/libdem.so smem6:$V/libdem_broad6.so; do
  tag=${L%%:*}; lib=${L#*:}
  DEM_LIB_VARIANT=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_broad --csv \
    --log-file gpurun_out/broad46_$tag.csv python profiles/rebuild_timing.py --n 12 --tag $tag > gpurun_out/broad46_$tag.log 2>&1
  tail -1 gpurun_out/broad46_$tag.log | cut -c1-200
done
