for V in 1 0; do
  echo "=== GJ_K2_VARIANT=$V"
  export GJ_K2_VARIANT=$V
  timeout 600 python -m pytest tests/test_gpu_batched.py -q -x -k "c3 or 64 or singular or det or hadamard or perm or in_place or host" 2>&1 | tail -2
  timeout 300 python tools/time_batched.py c3 2>&1 | tail -1
done
