# round 2, GPU call 19: coalesced tile staging (consecutive threads take consecutive 16-B chunks) vs the per-particle staging (g0 old); L1 prefetch variant on the new staging (g2)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python profiles/sweep_ab.py --tag stage_coal > gpurun_out/ab19.jsonl 2> gpurun_out/ab19.err
DEM_LIB_VARIANT=$V/libdem_g0.so timeout 300 python profiles/sweep_ab.py --tag stage_old >> gpurun_out/ab19.jsonl 2>> gpurun_out/ab19.err
DEM_LIB_VARIANT=$V/libdem_g2.so timeout 300 python profiles/sweep_ab.py --tag stage_coal_g2 >> gpurun_out/ab19.jsonl 2>> gpurun_out/ab19.err
cat gpurun_out/ab19.jsonl
