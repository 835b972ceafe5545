#!/bin/bash
# rns_kernel 128-byte stages (in-tree lib, 6 stages) vs 256-byte stages (abvar/lib256.so, 3 stages):
# short K halves the stage handshakes per pass
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in 1 2; do for L in paper_2601_07508_b200/libfpmm_b200.so abvar/lib256.so; do
  for shape in "40 16384 256 16384" "20 16384 256 16384" "52 16384 256 16384" "40 8192 512 8192" "20 8192 8192 8192" "52 8192 8192 8192"; do
    echo "$L $shape: $(FPMM_B200_LIB=$L FPMM_B200_RNS_TILE=0 ENGINE=rns timeout 120 python tools/one_product.py $shape 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
  done
done; done
