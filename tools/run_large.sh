# large-n path: parity tests + timing
timeout 900 python -m pytest tests/test_gpu_large.py -q -x 2>&1 | tail -4
timeout 300 python tools/time_large.py 2048 4096 8192 2>&1 | tail -4
