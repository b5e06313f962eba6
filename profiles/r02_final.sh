# round 2, final evidence (re-run after the own-particle select): bench lines (config4-geom with plates; config4-count), the launch list of
# the bench's timed window and one ncu --set full capture of k_sweep inside it (TMA-staged kernel)
set -x
mkdir -p gpurun_out
nproc
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; cat gpurun_out/bench_final2.json; tail -3 gpurun_out/bench_final2.err
timeout 1500 python bench.py --workload config4-count --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_count2.json 2> gpurun_out/bench_count2.err; cat gpurun_out/bench_count2.json; tail -3 gpurun_out/bench_count2.err
timeout 600 python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/bench_profile4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 5000 -c 3000 --csv --log-file gpurun_out/launches_timed2.csv \
    python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/ncu_launch3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1850 -c 1 -o gpurun_out/prof_bench_sweep_timed2 \
    python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/ncu_full3.log 2>&1
tail -2 gpurun_out/ncu_full3.log
