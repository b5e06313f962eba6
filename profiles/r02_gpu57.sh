# round 2, GPU call 57 (re-created container, library rebuilt from the unchanged round-2 sources):
# the driver's GPU tier, smoke, the default bench line, and one bench line of the decomposed path
# (NCCL transport, one rank) at the bench size
set -x
mkdir -p gpurun_out
nproc; nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout 1800 python -m pytest tests/ -x -q -m gpu -rxX -p no:cacheprovider > gpurun_out/gputests57.log 2>&1; tail -6 gpurun_out/gputests57.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke57.log 2>&1; tail -2 gpurun_out/smoke57.log | cut -c1-400
timeout 900 python bench.py > gpurun_out/bench57.json 2> gpurun_out/bench57.err; cat gpurun_out/bench57.json; tail -3 gpurun_out/bench57.err
timeout 900 python bench.py --decompose --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench57_decomp.json 2> gpurun_out/bench57_decomp.err; cat gpurun_out/bench57_decomp.json; tail -3 gpurun_out/bench57_decomp.err
