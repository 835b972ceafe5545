#!/bin/bash
# pack_a_rns thread mapping: 8 rows x 4 k16 chunks per warp (0) vs 32 rows x 1 chunk (1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
FPMM_B200_RNS_PACKA_ROWS=1 timeout 300 python -m pytest tests/test_parity_rns_gpu.py -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for v in 0 1; do for shape in "52 8192 8192 8192" "20 8192 8192 8192" "48 4096 262144 4096"; do
  echo "rows32=$v $shape: $(FPMM_B200_RNS_PACKA_ROWS=$v ENGINE=rns timeout 120 python tools/one_product.py $shape 5 | tail -1 | grep -o "pack_ms.: [0-9.]*")"
done; done; done
