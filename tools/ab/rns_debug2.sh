#!/bin/bash
# short-K rns_kernel skeleton (FPMM_B200_RNS_DEBUG bits: 1 no stores, 2 no epilogue work,
# 4 no MMAs, 8 MMAs skip the drain wait, 16 no operand loads); 16384^2 x 256, 40 bits
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for D in ${DBG:-0 2 6 22 30 0}; do
  echo "debug=$D: $(FPMM_B200_RNS_DEBUG=$D ENGINE=rns timeout 120 python tools/one_product.py 40 16384 256 16384 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*" | tr '\n' ' ')"
done
