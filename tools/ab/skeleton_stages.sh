#!/bin/bash
# rns_kernel barrier skeleton (FPMM_B200_RNS_DEBUG=22: no loads, no MMAs, no epilogue work) and full
# runs with 6 x 128-byte stages (in-tree lib) vs 12 x 64-byte stages (abvar/lib64.so): is the per-stage
# handshake bound by latency (time per stage halves with twice the stages in flight)?
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for L in paper_2601_07508_b200/libfpmm_b200.so abvar/lib64.so; do for D in 22 0; do
  for shape in "20 8192 8192 8192" "40 16384 256 16384"; do
    echo "$L debug=$D $shape: $(FPMM_B200_LIB=$L FPMM_B200_RNS_TILE=0 FPMM_B200_RNS_DEBUG=$D ENGINE=rns timeout 120 python tools/one_product.py $shape 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
  done
done; done
