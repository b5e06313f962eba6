# round 2, GPU call 23: ncu --set full of the shipped sweep (coalesced staging) on config4-geom
set -x
mkdir -p gpurun_out
timeout 300 python profiles/sweep_ab.py --tag pre_ncu --n 2 > gpurun_out/ab23.jsonl 2> gpurun_out/ab23.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1500 -c 1 -o gpurun_out/prof_sweep_r02f \
    python profiles/sweep_ab.py --tag ncu --n 2 > gpurun_out/ncu23.log 2>&1
tail -3 gpurun_out/ncu23.log
