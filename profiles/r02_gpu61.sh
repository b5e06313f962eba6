# round 2, GPU call 61: the final tree (sweep.cu with the SWEEP_SIG16 option off): the driver's GPU
# tier, smoke, and a short bench line
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -x -q -m gpu -rxX -p no:cacheprovider > gpurun_out/gputests61.log 2>&1; tail -5 gpurun_out/gputests61.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke61.log 2>&1; tail -1 gpurun_out/smoke61.log | cut -c1-300
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench61.json 2> gpurun_out/bench61.err; cut -c1-300 gpurun_out/bench61.json
