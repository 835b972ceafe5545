#!/bin/bash
# CRT finalisation on the FP64 pipe for p <= 2^40 (in-tree) vs the integer one-reduction form (abvar/libfinold.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests/test_parity_rns_gpu.py tests/test_fullsize_gpu.py -m gpu -x -q 2>&1 | tail -1
FPMM_B200_RNS_TILE=1 timeout 300 python tools/tile_check.py quick 2>&1 | tail -1
for r in 1 2; do for L in paper_2601_07508_b200/libfpmm_b200.so abvar/libfinold.so; do
  for shape in "40 65536 256 65536" "40 16384 256 16384" "20 16384 256 16384" "36 8192 8192 8192" "40 8192 8192 8192" "24 8192 8192 8192"; do
    echo "$L $shape: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py $shape 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*\|recon_ms.: [0-9.]*" | tr '\n' ' ')"
  done
done; done
