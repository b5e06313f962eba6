# ncu --set full of the sweep-kernel variants on config3-geom (run from the repo root under gpurun)
set -x
C1="python profiles/sweep_variants.py --workload config3-geom --variants ${VARIANTS:-0,10,20} --n 2 --settle 5"
$C1 > gpurun_out/plain.log 2>&1 || exit 1
for K in ${KERNELS:-k_sweep6 k_sweep5_ppt}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/prof_$K $C1 > gpurun_out/ncu_$K.log 2>&1
done
