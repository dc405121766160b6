# Round-2 profile set (run under gpurun after the same commands exited 0 without ncu):
#  1. launch list of the headline bench command (serialised, cold-cache per-launch times)
#  2. ncu --set full of K4b (one trailing update of the C4 inversion)
#  3. ncu --set full of K2f (C3-shaped batch)
set -e
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c2_launches.csv \
    python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-c4 > gpurun_out/r02_c2_launch.log 2>&1
bash tools/prof_dgemm.sh
bash tools/prof_k2e.sh
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c4_launches.csv \
    python tools/profile_large_once.py 8192 > /dev/null 2>&1
