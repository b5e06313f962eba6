# round 2, GPU call 8: tile 256 vs 128 (4 CTAs/SM) vs halo staging, with precomputed warp ranges
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python profiles/sweep_ab.py --tag tt256 > gpurun_out/ab8.jsonl 2> gpurun_out/ab8.err
DEM_LIB_VARIANT=$V/libdem_tt128.so timeout 300 python profiles/sweep_ab.py --tag tt128 >> gpurun_out/ab8.jsonl 2>> gpurun_out/ab8.err
DEM_LIB_VARIANT=$V/libdem_halo.so timeout 300 python profiles/sweep_ab.py --tag halo448 >> gpurun_out/ab8.jsonl 2>> gpurun_out/ab8.err
cat gpurun_out/ab8.jsonl; tail -2 gpurun_out/ab8.err
DEM_LIB_VARIANT=$V/libdem_tt128.so timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_column.py -q -x -p no:cacheprovider -k "chaotic or one_step" > gpurun_out/t8.log 2>&1; tail -2 gpurun_out/t8.log
