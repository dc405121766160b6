# one gpurun call: parity tests, smoke, bench line, ncu launch list, large-n timing
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 50 --warmup 3 --e2e-steps 2 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 300 python tools/time_large.py 4096 8192 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?
