# round 2, GPU call 22: c1-mini curves, seed-averaged bar, GPU curves saved
set -x
mkdir -p gpurun_out
nproc
timeout 2400 python -m pytest tests/test_gpu_curves_mini.py -q -x -p no:cacheprovider -k c1 -s > gpurun_out/t22.log 2>&1; tail -12 gpurun_out/t22.log
