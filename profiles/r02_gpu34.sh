# round 2, GPU call 34: compute-sanitizer memcheck / racecheck / synccheck of the shipped kernels (TMA staging, ragged odd last tile)
set -x
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $S --tool memcheck --leak-check no python profiles/sanitize_run.py 1501 > gpurun_out/san_mem.log 2>&1; tail -4 gpurun_out/san_mem.log
timeout 1200 $S --tool racecheck --racecheck-report hazard python profiles/sanitize_run.py 1501 > gpurun_out/san_race.log 2>&1; tail -4 gpurun_out/san_race.log
timeout 900 $S --tool synccheck python profiles/sanitize_run.py 1501 > gpurun_out/san_sync.log 2>&1; tail -4 gpurun_out/san_sync.log
timeout 900 $S --tool initcheck python profiles/sanitize_run.py 1501 > gpurun_out/san_init.log 2>&1; tail -4 gpurun_out/san_init.log
