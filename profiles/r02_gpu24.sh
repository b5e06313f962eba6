# round 2, GPU call 24: tile staging by TMA bulk copies on an mbarrier (default) vs per-thread cp.async (tma0)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python profiles/sweep_ab.py --tag tma > gpurun_out/ab24.jsonl 2> gpurun_out/ab24.err
DEM_LIB_VARIANT=$V/libdem_tma0.so timeout 300 python profiles/sweep_ab.py --tag tma0 >> gpurun_out/ab24.jsonl 2>> gpurun_out/ab24.err
cat gpurun_out/ab24.jsonl; tail -3 gpurun_out/ab24.err
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_column.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/t24.log 2>&1; tail -3 gpurun_out/t24.log
