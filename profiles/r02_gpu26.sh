# round 2, GPU call 26: contact arrays sized by the contact count (not the candidates): GPU suite + bench memory
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_curves_mini.py > gpurun_out/t26.log 2>&1; tail -3 gpurun_out/t26.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench26.json 2> gpurun_out/bench26.err; cat gpurun_out/bench26.json; tail -3 gpurun_out/bench26.err
