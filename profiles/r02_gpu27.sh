# round 2, GPU call 27: the rebuild permutes into the rollback buffers (no pos2/vel2/ang2): GPU suite + bench memory
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_curves_mini.py > gpurun_out/t27.log 2>&1; tail -3 gpurun_out/t27.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench27.json 2> gpurun_out/bench27.err; cat gpurun_out/bench27.json; tail -3 gpurun_out/bench27.err
