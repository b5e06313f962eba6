# round 2, GPU call 7: halo-staged cross partners
set -x
mkdir -p gpurun_out
timeout 300 python profiles/sweep_ab.py --tag v7halo > gpurun_out/ab7.jsonl 2> gpurun_out/ab7.err; cat gpurun_out/ab7.jsonl; tail -2 gpurun_out/ab7.err
timeout 300 python profiles/sweep_ab.py --tag v7 --n 20 > gpurun_out/ab7_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 8 -c 1 -o gpurun_out/prof_sweep_r02d \
   python profiles/sweep_ab.py --tag v7 --n 20 > gpurun_out/ncu_d.log 2>&1
tail -1 gpurun_out/ncu_d.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_curves_mini.py > gpurun_out/gpu_tests7.log 2>&1; tail -8 gpurun_out/gpu_tests7.log
