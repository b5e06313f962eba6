# round 2, GPU call 30: cross-tile partner loads issued before the segment set-up (early, default) vs inside the item branch (late)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python profiles/sweep_ab.py --tag early > gpurun_out/ab30.jsonl 2> gpurun_out/ab30.err
DEM_LIB_VARIANT=$V/libdem_late.so timeout 300 python profiles/sweep_ab.py --tag late >> gpurun_out/ab30.jsonl 2>> gpurun_out/ab30.err
timeout 300 python profiles/sweep_ab.py --tag early_again >> gpurun_out/ab30.jsonl 2>> gpurun_out/ab30.err
cat gpurun_out/ab30.jsonl; tail -3 gpurun_out/ab30.err
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_column.py -q -x -p no:cacheprovider > gpurun_out/t30.log 2>&1; tail -3 gpurun_out/t30.log
