# ncu --set full capture of the fp32 n=32 kernel on the C2 bench command
CMD="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-gj_blk32} -s 3 -c 1 -o gpurun_out/${OUT:-prof_k1b} $CMD > gpurun_out/ncu.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu.log
