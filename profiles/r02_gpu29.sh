# round 2, GPU call 29: own particle of cross items from smem (own) and L1::no_allocate record loads (nol1): both (default), base, own, nol1
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python profiles/sweep_ab.py --tag own+nol1 > gpurun_out/ab29.jsonl 2> gpurun_out/ab29.err
for t in base own nol1; do DEM_LIB_VARIANT=$V/libdem_$t.so timeout 300 python profiles/sweep_ab.py --tag $t >> gpurun_out/ab29.jsonl 2>> gpurun_out/ab29.err; done
cat gpurun_out/ab29.jsonl; tail -3 gpurun_out/ab29.err
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_column.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/t29.log 2>&1; tail -3 gpurun_out/t29.log
