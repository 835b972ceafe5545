#!/bin/bash
# RNS rasterisation group on the 8192^3 sweep (pair-tile rows per group; MB = 32 at 8192)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in 1 2; do for G in 16 32 8; do
  echo "group=$G: $(FPMM_B200_RNS_GROUP=$G timeout 300 python bench.py --no-e2e --no-cpu --no-engines --steps 5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], d["roofline"]["achieved"])')"
done; done
