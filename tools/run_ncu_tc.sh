python tools/profile_large_f32_once.py 8192 > gpurun_out/p32.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f32_launches.csv python tools/profile_large_f32_once.py 8192 > gpurun_out/ncu32.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_update -s 20 -c 1 -o gpurun_out/prof_tc python tools/profile_large_f32_once.py 8192 > gpurun_out/ncu_tc.log 2>&1; echo rc=$?
