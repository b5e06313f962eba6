# round 2, GPU call 54: the driver's round-end GPU tier on the final tree: pytest -m gpu (all GPU tests,
# the curve acceptance last) and smoke()
set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider -rxX > gpurun_out/gpu_all54.log 2>&1; tail -8 gpurun_out/gpu_all54.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke54.log 2>&1; tail -1 gpurun_out/smoke54.log | cut -c1-120
