#!/bin/bash
# A/B of library builds on the bench's timed sweep (same box, alternating):
#   LIBS="abvar/a.so abvar/b.so" bash tools/ab/ab_bench_libs.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in ${ROUNDS:-1 2}; do for L in ${LIBS}; do
  FPMM_B200_LIB=$L timeout 400 python bench.py --no-e2e --no-cpu --no-engines --steps 5 > gpurun_out/ab_bench.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab_bench.json').read().strip().splitlines()[-1])
print('$L', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['frac'])"
done; done
