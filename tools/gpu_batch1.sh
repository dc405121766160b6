set -x
mkdir -p gpurun_out
timeout 600 python tools/fuzz_find_g27_case.py 7 8 > gpurun_out/g27find.log 2>&1
timeout 900 python -m pytest tests/test_gpu_precision_ladder.py -q -s 2>&1 | grep -E "max e|passed|failed" > gpurun_out/ladder.log
timeout 900 python -m pytest tests/test_gpu_batched_sharded.py tests/test_gpu_dist.py -q -x > gpurun_out/shard_dist.log 2>&1
GJ_PARITY_REPORT=gpurun_out/c2_parity.json timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c2_every_item" > gpurun_out/c2every.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
tail -3 gpurun_out/*.log
