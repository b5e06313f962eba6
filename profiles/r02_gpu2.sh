# round 2, GPU call 2: sweep A/B (80-reg x3 CTAs vs 128-reg x2 CTAs), then the GPU suite
set -x
mkdir -p gpurun_out
timeout 300 python profiles/sweep_ab.py --tag minb3 > gpurun_out/ab.jsonl 2> gpurun_out/ab.err
DEM_LIB_VARIANT=paper_2501_05300_b200/lib/variants/libdem_minb2.so timeout 300 python profiles/sweep_ab.py --tag minb2 >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
cat gpurun_out/ab.jsonl; tail -3 gpurun_out/ab.err
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests2.log 2>&1; tail -25 gpurun_out/gpu_tests2.log
