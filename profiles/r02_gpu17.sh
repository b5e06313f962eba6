# round 2, GPU call 17: the cp.async partner ring with the shared-memory carveout at 100 % (occupancy printed)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
DEM_DEBUG=1 timeout 300 python profiles/sweep_ab.py --tag gather_c100 > gpurun_out/ab17.jsonl 2> gpurun_out/ab17.err
DEM_DEBUG=1 DEM_LIB_VARIANT=$V/libdem_g0.so timeout 300 python profiles/sweep_ab.py --tag g0_c100 >> gpurun_out/ab17.jsonl 2>> gpurun_out/ab17.err
cat gpurun_out/ab17.jsonl; grep "k_sweep:" gpurun_out/ab17.err
