#!/bin/bash
# rns_kernel MMA issuer: converged warp + elect.sync (in-tree) vs one thread (abvar/libthread.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 300 python -m pytest tests/test_parity_rns_gpu.py -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for L in paper_2601_07508_b200/libfpmm_b200.so abvar/libthread.so; do
  for shape in "40 16384 256 16384" "20 16384 256 16384" "52 16384 256 16384" "40 8192 1024 8192" "20 8192 8192 8192" "52 8192 8192 8192"; do
    echo "$L $shape: $(FPMM_B200_LIB=$L FPMM_B200_RNS_TILE=0 ENGINE=rns timeout 120 python tools/one_product.py $shape 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
  done
  echo "$L debug=22 40 16384 256 16384: $(FPMM_B200_LIB=$L FPMM_B200_RNS_DEBUG=22 FPMM_B200_RNS_TILE=0 ENGINE=rns timeout 120 python tools/one_product.py 40 16384 256 16384 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
done; done
