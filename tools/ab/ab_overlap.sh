#!/bin/bash
# RNS row-block pipeline (FPMM_B200_RNS_OVERLAP=<GEMM pairs>): GEMM of block b+1 beside the CRT of block b
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
FPMM_B200_RNS_OVERLAP=50 timeout 300 python -m pytest tests/test_fullsize_gpu.py -m gpu -x -q -k "row_blocks or c5 or c3_32768" 2>&1 | tail -1
for ov in 0 74 64 56 48 40; do
  FPMM_B200_RNS_OVERLAP=$ov timeout 300 python tools/bench_configs.py --only c5,c3 --engines rns --out gpurun_out/ov_$ov.json > /dev/null 2>&1
  python -c "
import json
for r in json.load(open('gpurun_out/ov_$ov.json')): print('overlap=$ov', r['m'], r['k'], r['n'], r['ms'], r['eff_gflops'])"
done
