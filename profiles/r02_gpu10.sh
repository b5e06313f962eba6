# round 2, GPU call 10: occupancy vs registers (prefetch on/off, tile 256/128)
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python profiles/sweep_ab.py --tag m2pf > gpurun_out/ab10.jsonl 2> gpurun_out/ab10.err
for v in m3pf m3np t128m6 t128m8np; do
  DEM_LIB_VARIANT=$V/libdem_$v.so timeout 300 python profiles/sweep_ab.py --tag $v >> gpurun_out/ab10.jsonl 2>> gpurun_out/ab10.err
done
cat gpurun_out/ab10.jsonl; tail -3 gpurun_out/ab10.err
