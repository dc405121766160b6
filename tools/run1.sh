set -x
python -m pytest tests -q -m gpu -x 2>&1 | tail -30
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
python bench.py --steps 50 --warmup 3 --e2e-steps 2 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo rc=$?
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
