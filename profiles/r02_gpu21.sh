# round 2, GPU call 21: c1-mini plate curves (3 seeds, 4e4 steps) GPU vs the stored oracle curves (re-run 22 with the seed-averaged bar)
set -x
mkdir -p gpurun_out
nproc
timeout 2400 python -m pytest tests/test_gpu_curves_mini.py -q -x -p no:cacheprovider -k c1 -s > gpurun_out/t21.log 2>&1; tail -12 gpurun_out/t21.log
