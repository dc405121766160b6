# A/B of the fp32 n=32 kernel variants: parity tests + bench for each (block size, stages)
for V in ${VARIANTS:-4:2 4:1 8:1}; do
  B=${V%%:*}; S=${V##*:}
  echo "=== GJ_K1_BLOCK=$B GJ_K1_STAGES=$S"
  GJ_K1_BLOCK=$B GJ_K1_STAGES=$S timeout 600 python -m pytest tests/test_gpu_batched.py -q -x 2>&1 | tail -2
  GJ_K1_BLOCK=$B GJ_K1_STAGES=$S timeout 300 python bench.py --steps 30 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], 'frac', d['roofline']['frac'], d['clocks'])"
done
