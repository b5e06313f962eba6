# round 2, GPU call 4: column parity for the impulse-storage variants and the round-1 kernel;
# ncu capture of the current sweep
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
for v in r1 minb2_p1 minb2_p2; do
  DEM_LIB_VARIANT=$V/libdem_$v.so timeout 900 python -m pytest tests/test_gpu_bench_column.py -q -s -p no:cacheprovider -k one_step > gpurun_out/col_$v.log 2>&1; echo "== $v"; grep -E "force_err|passed|failed" gpurun_out/col_$v.log | cut -c1-330
done
for v in r1 minb2_p1 minb2_p2; do
  DEM_LIB_VARIANT=$V/libdem_$v.so timeout 300 python profiles/sweep_ab.py --tag $v >> gpurun_out/ab4.jsonl 2>> gpurun_out/ab4.err
done
cat gpurun_out/ab4.jsonl
DEM_LIB_VARIANT=$V/libdem_minb2.so timeout 300 python profiles/sweep_ab.py --tag minb2 --n 20 > gpurun_out/ab4_plain.log 2>&1 && \
DEM_LIB_VARIANT=$V/libdem_minb2.so ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 8 -c 1 -o gpurun_out/prof_sweep_r02b \
   python profiles/sweep_ab.py --tag minb2 --n 20 > gpurun_out/ncu_b.log 2>&1
tail -2 gpurun_out/ncu_b.log
