# round 2, GPU call 5: fp64-impulse item layout: timing, ncu capture, parity suite
set -x
mkdir -p gpurun_out
timeout 300 python profiles/sweep_ab.py --tag fp64P > gpurun_out/ab5.jsonl 2> gpurun_out/ab5.err; cat gpurun_out/ab5.jsonl; tail -2 gpurun_out/ab5.err
timeout 300 python profiles/sweep_ab.py --tag fp64P --n 20 > gpurun_out/ab5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 8 -c 1 -o gpurun_out/prof_sweep_r02c \
   python profiles/sweep_ab.py --tag fp64P --n 20 > gpurun_out/ncu_c.log 2>&1
tail -1 gpurun_out/ncu_c.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests5.log 2>&1; tail -15 gpurun_out/gpu_tests5.log
