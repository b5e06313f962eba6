# round 2, GPU call 15: round-robin 32-item chunks per warp (SWEEP_RR=1) vs plan ranges (rr0)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python profiles/sweep_ab.py --tag rr1 > gpurun_out/ab15.jsonl 2> gpurun_out/ab15.err
DEM_LIB_VARIANT=$V/libdem_rr0.so timeout 300 python profiles/sweep_ab.py --tag rr0 >> gpurun_out/ab15.jsonl 2>> gpurun_out/ab15.err
cat gpurun_out/ab15.jsonl; tail -3 gpurun_out/ab15.err
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_column.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/t15.log 2>&1; tail -3 gpurun_out/t15.log
