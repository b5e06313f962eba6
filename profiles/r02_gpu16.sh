# round 2, GPU call 16: cross-tile partners gathered a chunk ahead by cp.async (SWEEP_GATHER=1) vs direct loads (g0)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python profiles/sweep_ab.py --tag gather > gpurun_out/ab16.jsonl 2> gpurun_out/ab16.err
DEM_LIB_VARIANT=$V/libdem_g0.so timeout 300 python profiles/sweep_ab.py --tag g0 >> gpurun_out/ab16.jsonl 2>> gpurun_out/ab16.err
cat gpurun_out/ab16.jsonl; tail -3 gpurun_out/ab16.err
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_column.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/t16.log 2>&1; tail -3 gpurun_out/t16.log
