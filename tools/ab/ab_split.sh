#!/bin/bash
# rns_kernel short K: accumulator column halves with their own MMAs and barriers (FPMM_B200_RNS_SPLIT=1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
FPMM_B200_RNS_SPLIT=1 FPMM_B200_RNS_TILE=0 timeout 300 python -m pytest tests/test_parity_rns_gpu.py tests/test_parity_gpu.py -m gpu -x -q -k "rns or RNS or default or None" 2>&1 | tail -1
FPMM_B200_RNS_SPLIT=1 FPMM_B200_RNS_TILE=0 timeout 300 python tools/tile_check.py quick 2>&1 | tail -1
for r in 1 2; do for v in 0 1; do
  for shape in "40 16384 256 16384" "20 16384 256 16384" "52 16384 256 16384" "40 8192 512 8192" "40 8192 1024 8192" "40 65536 256 65536"; do
    echo "split=$v $shape: $(FPMM_B200_RNS_SPLIT=$v FPMM_B200_RNS_TILE=0 ENGINE=rns timeout 120 python tools/one_product.py $shape 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
  done
done; done
