# round-end evidence: ncu --set full of the default K1 (C2 bench command), the bench launch
# list, and one panel + one trailing GEMM of the C4 path
set -x
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-c4"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gj_blk32 -s 3 -c 1 -o gpurun_out/prof_k1_final $CMD > gpurun_out/ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu2.log 2>&1
python tools/profile_large_once.py 8192 > gpurun_out/plain_large.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:leaf_kernel -s 5 -c 1 -o gpurun_out/prof_panel python tools/profile_large_once.py 8192 > gpurun_out/ncu3.log 2>&1
echo done
