#!/bin/bash
# C3 / C4 rasterisation group (pair-tile rows per group) and pacing window (256-byte k-blocks)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for cfg in "16 32" "12 32" "20 32" "24 32" "16 16" "16 64"; do
  set -- $cfg
  FPMM_B200_RNS_GROUP=$1 FPMM_B200_RNS_PACE=$2 timeout 300 python tools/bench_configs.py --only c3,c4 --engines rns --out gpurun_out/g_$1_$2.json > /dev/null 2>&1
  python -c "
import json
for r in json.load(open('gpurun_out/g_$1_$2.json')): print('group=$1 pace=$2', r['m'], r['k'], r['n'], r['ms'], r['eff_gflops'], r['gemm_ms'])"
done
