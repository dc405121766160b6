# ncu of the f2 (K6) and f4 (K7) kernels on C2-sized batches
python tools/profile_f2_f4_once.py || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f2f4_launches.csv python tools/profile_f2_f4_once.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gj_full_kernel|gj_solve_kernel" -c 2 -o gpurun_out/f2f4 python tools/profile_f2_f4_once.py > gpurun_out/f2f4_ncu.log 2>&1
tail -2 gpurun_out/f2f4_ncu.log
