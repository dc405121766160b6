python tools/profile_large_once.py 8192 > gpurun_out/plain_large.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_update --launch-skip 21 -c 1 -o gpurun_out/prof_gemm python tools/profile_large_once.py 8192 > gpurun_out/ncu_gemm.log 2>&1; echo rc=$?
