# round 2, GPU call 53: c2-mini plate curves (3 seeds, 5e4 steps, monolithic plate coupling) against the
# regenerated oracle curves, from the cached oracle-settled beds; c1-mini again
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_z_curves_mini.py -q -s -p no:cacheprovider > gpurun_out/curves53.log 2>&1; grep -E "rms|passed|failed|Error" gpurun_out/curves53.log | tail -12
