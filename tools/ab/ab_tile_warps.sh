#!/bin/bash
# rns_tile_kernel epilogue: 16 warps x 32 columns (in-tree) vs 8 warps x 64 columns (abvar/libtile8.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
FPMM_B200_LIB=abvar/libtile8.so FPMM_B200_RNS_TILE=1 timeout 300 python tools/tile_check.py quick 2>&1 | tail -1
for r in 1 2; do for L in paper_2601_07508_b200/libfpmm_b200.so abvar/libtile8.so; do
  for shape in "40 65536 256 65536" "40 16384 256 16384" "20 16384 256 16384" "30 16384 256 16384"; do
    echo "$L $shape: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py $shape 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
  done
done; done
