# round 2, GPU call 20: the cleaned sweep (coalesced staging, no ring/prefetch/round-robin options): timing + parity
set -x
mkdir -p gpurun_out
timeout 300 python profiles/sweep_ab.py --tag clean > gpurun_out/ab20.jsonl 2> gpurun_out/ab20.err
cat gpurun_out/ab20.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_curves_mini.py > gpurun_out/t20.log 2>&1; tail -3 gpurun_out/t20.log
