python tools/profile_large_once.py ${N:-8192} > gpurun_out/plain_large.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/large_launches.csv python tools/profile_large_once.py ${N:-8192} > gpurun_out/ncu_large.log 2>&1; echo rc=$?
