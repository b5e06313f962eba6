# round 2, GPU call 9: persistent CTAs with cp.async double-buffered tile staging
set -x
mkdir -p gpurun_out
timeout 300 python profiles/sweep_ab.py --tag persist > gpurun_out/ab9.jsonl 2> gpurun_out/ab9.err; cat gpurun_out/ab9.jsonl; tail -2 gpurun_out/ab9.err
timeout 300 python profiles/sweep_ab.py --tag persist --n 20 > gpurun_out/ab9_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 8 -c 1 -o gpurun_out/prof_sweep_r02e \
   python profiles/sweep_ab.py --tag persist --n 20 > gpurun_out/ncu_e.log 2>&1
tail -1 gpurun_out/ncu_e.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_curves_mini.py > gpurun_out/gpu_tests9.log 2>&1; tail -8 gpurun_out/gpu_tests9.log
