#!/bin/bash
# short-K rns_kernel: pingpong drain with one (0) or two (1) 32-column TMEM loads per wait
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for rep in 1 2; do for v in 0 1; do
  for shape in "40 16384 256 16384" "20 16384 256 16384" "52 16384 256 16384" "40 8192 1024 8192"; do
    echo "pp_pairs=$v $shape: $(FPMM_B200_RNS_TILE=0 FPMM_B200_RNS_PP_PAIRS=$v ENGINE=rns timeout 120 python tools/one_product.py $shape 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
  done
done; done
