#!/bin/bash
# 256-byte RNS stages (abvar/lib256.so): GPU tests, BASELINE configs and the sweep against the in-tree lib
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
FPMM_B200_LIB=abvar/lib256.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest256.log 2>&1; tail -2 gpurun_out/pytest256.log
for L in paper_2601_07508_b200/libfpmm_b200.so abvar/lib256.so; do
  FPMM_B200_LIB=$L timeout 600 python tools/bench_configs.py --only c3,c4,c5 --engines rns --out gpurun_out/cfg_$(basename $L .so).json > /dev/null 2>&1
  echo "$L sweep: $(FPMM_B200_LIB=$L timeout 300 python bench.py --no-e2e --no-cpu --no-engines --steps 5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], d["roofline"]["achieved"])')"
done
