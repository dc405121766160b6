set -x
python -m pytest tests -q -m gpu -x 2>&1 | tail -30
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py --steps 100 --warmup 5 --e2e-steps 2 > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo rc=$?
cat gpurun_out/bench8.json; tail -3 gpurun_out/bench8.err
python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gj_batched -s 3 -c 1 -o gpurun_out/prof_k1g \
  python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu.log
