# round 2, GPU call 28: chunk loop unrolled twice (two record register sets, default) vs one (u1)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python profiles/sweep_ab.py --tag unroll2 > gpurun_out/ab28.jsonl 2> gpurun_out/ab28.err
DEM_LIB_VARIANT=$V/libdem_u1.so timeout 300 python profiles/sweep_ab.py --tag unroll1 >> gpurun_out/ab28.jsonl 2>> gpurun_out/ab28.err
cat gpurun_out/ab28.jsonl; tail -3 gpurun_out/ab28.err
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_column.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/t28.log 2>&1; tail -3 gpurun_out/t28.log
