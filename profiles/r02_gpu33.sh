# round 2, GPU call 33: more warps per SM: 192-particle tiles x 3 CTAs (18 warps, 96 regs) and 160 x 4 (20 warps, 96 regs) vs the shipped 256 x 2
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
DEM_DEBUG=1 timeout 300 python profiles/sweep_ab.py --tag t256 > gpurun_out/ab33.jsonl 2> gpurun_out/ab33.err
for t in t192 t160; do DEM_DEBUG=1 DEM_LIB_VARIANT=$V/libdem_$t.so timeout 300 python profiles/sweep_ab.py --tag $t >> gpurun_out/ab33.jsonl 2>> gpurun_out/ab33.err; done
cat gpurun_out/ab33.jsonl; grep "k_sweep:" gpurun_out/ab33.err
