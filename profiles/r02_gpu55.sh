# round 2, GPU call 55: bench lines of the round-2 library on the other SURVEY §8(d) workloads
# (config 1, 2, 3 in the stated geometry and the count variants), 3 timed steps each
set -x
mkdir -p gpurun_out
for w in config1 config2-geom config2-count config3-geom config3-count; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench55_$w.json 2> gpurun_out/bench55_$w.err
  tail -1 gpurun_out/bench55_$w.json | cut -c1-200; tail -1 gpurun_out/bench55_$w.err | cut -c1-200
done
