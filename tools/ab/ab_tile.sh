#!/bin/bash
# rns_tile_kernel stage-count A/B on the short-K shapes (tools/tile_check.py short)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for st in ${STAGES:-4 6 8}; do
  echo "== stages $st" >> gpurun_out/ab_tile.log
  FPMM_B200_RNS_TILE_STAGES=$st timeout 300 python tools/tile_check.py ${WHICH:-short} >> gpurun_out/ab_tile.log 2>&1
done
tail -40 gpurun_out/ab_tile.log
