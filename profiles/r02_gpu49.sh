# round 2, GPU call 49: c1-mini plate curves (3 seeds, 4e4 steps) from the cached oracle-settled beds
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_z_curves_mini.py -k c1 -q -s -p no:cacheprovider > gpurun_out/curves49.log 2>&1; grep -E "rms|passed|failed" gpurun_out/curves49.log | tail -8
