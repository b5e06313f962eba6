# round 2, GPU call 6: owner-in-record segments, slot-major slots, wider fixed-point range
set -x
mkdir -p gpurun_out
timeout 300 python profiles/sweep_ab.py --tag v6 > gpurun_out/ab6.jsonl 2> gpurun_out/ab6.err; cat gpurun_out/ab6.jsonl; tail -2 gpurun_out/ab6.err
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_curves_mini.py > gpurun_out/gpu_tests6.log 2>&1; tail -8 gpurun_out/gpu_tests6.log
