# round 2, GPU call 18: cross-tile partners one chunk ahead -- prefetched into L1 (g2, default), cp.async ring (g1), none (g0)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
DEM_DEBUG=1 timeout 300 python profiles/sweep_ab.py --tag g2 > gpurun_out/ab18.jsonl 2> gpurun_out/ab18.err
DEM_DEBUG=1 DEM_LIB_VARIANT=$V/libdem_g0.so timeout 300 python profiles/sweep_ab.py --tag g0 >> gpurun_out/ab18.jsonl 2>> gpurun_out/ab18.err
DEM_DEBUG=1 DEM_LIB_VARIANT=$V/libdem_g1.so timeout 300 python profiles/sweep_ab.py --tag g1 >> gpurun_out/ab18.jsonl 2>> gpurun_out/ab18.err
cat gpurun_out/ab18.jsonl; grep "k_sweep:" gpurun_out/ab18.err
