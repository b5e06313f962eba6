# round 2, GPU call 36: persistent CTAs with the next tile staged by TMA while the current computes
# (SWEEP_PERSIST=1; 256- and 512-particle tiles) vs the shipped sweep, sustained ms per sweep on
# config4-geom (profiles/sweep_ab.py), plus the parity suite on the persistent build
set -x
mkdir -p gpurun_out
V=paper_2501_05300_b200/lib/variants
timeout 600 python profiles/sweep_ab.py --tag ship > gpurun_out/ab36.log 2>&1
DEM_LIB_VARIANT=$V/libdem_pers.so timeout 600 python profiles/sweep_ab.py --tag pers256 >> gpurun_out/ab36.log 2>&1
DEM_LIB_VARIANT=$V/libdem_pers512.so timeout 600 python profiles/sweep_ab.py --tag pers512 >> gpurun_out/ab36.log 2>&1
timeout 600 python profiles/sweep_ab.py --tag ship2 >> gpurun_out/ab36.log 2>&1
grep '^{' gpurun_out/ab36.log
DEM_LIB_VARIANT=$V/libdem_pers.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_column.py -q -x -p no:cacheprovider > gpurun_out/pers_tests.log 2>&1; tail -3 gpurun_out/pers_tests.log
