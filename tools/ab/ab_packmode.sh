#!/bin/bash
# RNS packers by residue form (FPMM_B200_RNS_PACK_FP64: 0 digits/dp4a, 1 FP64 pairs, 2 integer pairs)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in 1 2; do for M in 0 1 2; do
  for shape in "52 8192 8192 8192" "36 8192 8192 8192" "20 8192 8192 8192" "48 4096 262144 4096"; do
    echo "mode=$M $shape: $(FPMM_B200_RNS_PACK_FP64=$M ENGINE=rns timeout 120 python tools/one_product.py $shape 3 | tail -1 | grep -o "pack_ms.: [0-9.]*")"
  done
done; done
timeout 300 python -m pytest tests/test_parity_rns_gpu.py -m gpu -x -q 2>&1 | tail -1
FPMM_B200_RNS_PACK_FP64=2 timeout 300 python -m pytest tests/test_parity_rns_gpu.py tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -1
