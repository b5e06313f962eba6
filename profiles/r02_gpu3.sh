# round 2, GPU call 3: sweep timings (round-1 kernel vs contact-once variants), column parity for both
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
DEM_LIB_VARIANT=$V/libdem_r1.so timeout 300 python profiles/sweep_ab.py --tag r1 > gpurun_out/ab3.jsonl 2> gpurun_out/ab3.err
timeout 300 python profiles/sweep_ab.py --tag minb3 >> gpurun_out/ab3.jsonl 2>> gpurun_out/ab3.err
DEM_LIB_VARIANT=$V/libdem_minb2.so timeout 300 python profiles/sweep_ab.py --tag minb2 >> gpurun_out/ab3.jsonl 2>> gpurun_out/ab3.err
cat gpurun_out/ab3.jsonl; tail -3 gpurun_out/ab3.err
DEM_LIB_VARIANT=$V/libdem_r1.so timeout 900 python -m pytest tests/test_gpu_bench_column.py -q -s -p no:cacheprovider -k one_step > gpurun_out/col_r1.log 2>&1; grep -E "force_err|passed|failed" gpurun_out/col_r1.log | cut -c1-400
timeout 900 python -m pytest tests/test_gpu_bench_column.py tests/test_gpu_parity.py tests/test_gpu_dist.py -q -s -p no:cacheprovider > gpurun_out/col_new.log 2>&1; grep -E "force_err|passed|failed" gpurun_out/col_new.log | cut -c1-400
