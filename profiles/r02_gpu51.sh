# round 2, GPU call 51: decomposed sweep loop captured in a CUDA graph with the halo exchange
# (grouped NCCL send/recv) inside (DEM_GRAPH_NCCL=1) -- one-rank NCCL self-test bit-identical to
# the single context; the whole decomposition suite
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/dist51.log 2>&1; tail -3 gpurun_out/dist51.log
