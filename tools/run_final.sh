# round-end style validation: all GPU tests, smoke, the bench line, the reference arm, the C5
# line, ncu launch lists (C2 bench command, C4) and the K1f ncu capture
set -x
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 900 python bench.py --workload c5 --steps 2 --warmup 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c2_launches.csv \
    python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-c4 > /dev/null 2>&1; echo ncu_c2_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c4_launches.csv \
    python tools/profile_large_once.py 8192 > /dev/null 2>&1; echo ncu_c4_rc=$?
bash tools/prof_k1b.sh > gpurun_out/prof_k1f.log 2>&1; echo prof_k1f_rc=$?
