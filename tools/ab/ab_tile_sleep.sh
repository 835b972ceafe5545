#!/bin/bash
# rns_tile_kernel: producer / MMA-warp waits polling with a sleep (FPMM_B200_RNS_TILE_SLEEP ns) vs spinning
cd "${GRAFT_REPO_ROOT:-/root/repo}"
FPMM_B200_RNS_TILE_SLEEP=64 FPMM_B200_RNS_TILE=1 timeout 300 python tools/tile_check.py quick 2>&1 | tail -1
for r in 1 2; do for ns in 0 32 128 512; do
  for shape in "40 65536 256 65536" "40 16384 256 16384" "20 16384 256 16384"; do
    echo "sleep=$ns $shape: $(FPMM_B200_RNS_TILE_SLEEP=$ns ENGINE=rns timeout 120 python tools/one_product.py $shape 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
  done
done; done
