python tools/time_batched.py c3 > gpurun_out/plain_k2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gj_batched64b -s 2 -c 1 -o gpurun_out/prof_k2b python tools/time_batched.py c3 > gpurun_out/ncu_k2.log 2>&1; echo rc=$?
