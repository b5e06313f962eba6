# round 2, GPU call 40: ncu --set full with source of one shipped k_sweep<false> launch on config4-geom
# (profiles/sweep_ab.py after its preparation), for the per-line stall breakdown
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep --launch-skip 30 --launch-count 1 \
  -o gpurun_out/sweep_src40 -f python profiles/sweep_ab.py --n 3 --settle 10 > gpurun_out/ncu40.log 2>&1
tail -3 gpurun_out/ncu40.log
ls -la gpurun_out/
