# round 2: launch list and full capture of the sweep inside the bench's TIMED window
set -x
mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread"
timeout 600 python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/bench_profile3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 5000 -c 3000 --csv --log-file gpurun_out/launches_timed.csv \
    python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/ncu_launch2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1850 -c 1 -o gpurun_out/prof_bench_sweep_timed \
    python bench.py --steps 1 --warmup 1 --settle 2 --profile > gpurun_out/ncu_full2.log 2>&1
tail -2 gpurun_out/ncu_full2.log
