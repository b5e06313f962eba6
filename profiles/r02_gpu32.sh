# round 2, GPU call 32: v/w halves de-interleaved by 2-D TMA tensor copies (default) vs 1-D bulk AoS staging (tma1)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python profiles/sweep_ab.py --tag tma2 > gpurun_out/ab32.jsonl 2> gpurun_out/ab32.err
DEM_LIB_VARIANT=$V/libdem_tma1.so timeout 300 python profiles/sweep_ab.py --tag tma1 >> gpurun_out/ab32.jsonl 2>> gpurun_out/ab32.err
cat gpurun_out/ab32.jsonl; tail -3 gpurun_out/ab32.err
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_column.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/t32.log 2>&1; tail -3 gpurun_out/t32.log
