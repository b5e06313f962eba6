# round 2, GPU call 13: timing experiments on the shipped sweep (wrong results): no scan, no conversion
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 300 python profiles/sweep_ab.py --tag shipped > gpurun_out/ab13.jsonl 2> gpurun_out/ab13.err
for v in noscan noconv; do
  DEM_LIB_VARIANT=$V/libdem_$v.so timeout 300 python profiles/sweep_ab.py --tag $v >> gpurun_out/ab13.jsonl 2>> gpurun_out/ab13.err
done
cat gpurun_out/ab13.jsonl; tail -3 gpurun_out/ab13.err
