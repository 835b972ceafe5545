# A/B of two library builds on the bench's timed sweep (same box, alternating)
for r in 1 2; do for L in abvar/lib8.so abvar/lib192.so; do
  FPMM_B200_LIB=$L timeout 400 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/ab_bench.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab_bench.json').read().strip().splitlines()[-1])
print('$L', d['value'], d['clocks']['sm_mhz'], d['roofline']['frac'])"
done; done
