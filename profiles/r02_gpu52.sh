# round 2, GPU call 52: bench line of the final round-2 library (config4-geom with the C21 plates)
set -x
mkdir -p gpurun_out
nproc
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench52.json 2> gpurun_out/bench52.err; cat gpurun_out/bench52.json; tail -3 gpurun_out/bench52.err
