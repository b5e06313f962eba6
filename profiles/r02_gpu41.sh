# round 2, GPU call 41: ncu --set full with source of one shipped main-stage k_sweep<false> launch on
# config4-geom (profiles/sweep_ab.py after its preparation), for the per-line stall breakdown
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_sweep<\(bool\)0' --launch-skip 25 --launch-count 1 \
  -o gpurun_out/sweep_src41 -f python profiles/sweep_ab.py --n 3 --settle 10 > gpurun_out/ncu41.log 2>&1
tail -3 gpurun_out/ncu41.log
