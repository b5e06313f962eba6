# round 2, GPU call 25: c2-mini curves (seed-averaged bar) + the whole GPU suite after the memory trim (Pa/Pb[1] and GS buffers)
set -x
mkdir -p gpurun_out
nproc
timeout 2400 python -m pytest tests/test_gpu_curves_mini.py -q -x -p no:cacheprovider -k c2 -s > gpurun_out/t25c.log 2>&1; grep rms gpurun_out/t25c.log; tail -2 gpurun_out/t25c.log
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_curves_mini.py > gpurun_out/t25.log 2>&1; tail -3 gpurun_out/t25.log
