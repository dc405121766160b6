# A/B of the fp32 n=32 kernel variants: parity tests + bench for each (rows/lane, block size, stages)
for V in ${VARIANTS:-2:4:2 4:4:1 4:8:1}; do
  R=${V%%:*}; rest=${V#*:}; B=${rest%%:*}; S=${rest##*:}
  echo "=== GJ_K1_ROWS=$R GJ_K1_BLOCK=$B GJ_K1_STAGES=$S"
  export GJ_K1_ROWS=$R GJ_K1_BLOCK=$B GJ_K1_STAGES=$S
  timeout 600 python -m pytest tests/test_gpu_batched.py -q -x 2>&1 | tail -2
  timeout 300 python bench.py --steps 30 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-c4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], 'frac', d['roofline']['frac'], d['clocks'])"
done
