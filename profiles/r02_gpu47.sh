# round 2, GPU call 47: smem-staged warp broad phase, staging capacity vs occupancy (k_broad ncu launch list)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
for tag in 128_8 96_10 64_12; do
  DEM_LIB_VARIANT=$V/libdem_broad_$tag.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_broad --csv \
    --log-file gpurun_out/broad47_$tag.csv python profiles/rebuild_timing.py --n 12 --tag $tag > gpurun_out/broad47_$tag.log 2>&1
  tail -1 gpurun_out/broad47_$tag.log | cut -c1-100
done
