#!/bin/bash
# rns_tile_kernel with 256-byte stages: stage count vs accumulators (FPMM_B200_RNS_TILE_STAGES; the host keeps >= 2 accumulators)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for st in 4 3 2; do for shape in "40 65536 256 65536" "40 16384 256 16384" "20 16384 256 16384" "30 16384 256 16384"; do
  echo "stages<=$st $shape: $(FPMM_B200_RNS_TILE=1 FPMM_B200_RNS_TILE_STAGES=$st ENGINE=rns timeout 120 python tools/one_product.py $shape 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
done; done
