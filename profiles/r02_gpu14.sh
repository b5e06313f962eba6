# round 2, GPU call 14: 512-particle tiles (one CTA of 16 warps per SM)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python profiles/sweep_ab.py --tag t256 > gpurun_out/ab14.jsonl 2> gpurun_out/ab14.err
DEM_LIB_VARIANT=$V/libdem_t512.so timeout 300 python profiles/sweep_ab.py --tag t512 >> gpurun_out/ab14.jsonl 2>> gpurun_out/ab14.err
cat gpurun_out/ab14.jsonl; tail -3 gpurun_out/ab14.err
DEM_LIB_VARIANT=$V/libdem_t512.so timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_column.py -q -x -p no:cacheprovider -k "chaotic or one_step" > gpurun_out/t14.log 2>&1; tail -2 gpurun_out/t14.log
