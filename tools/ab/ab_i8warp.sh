#!/bin/bash
# mwi8_kernel MMA issuer: converged warp + elect.sync (in-tree) vs lane 0 alone (abvar/libi8old.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 300 python -m pytest tests/test_parity_i8_gpu.py tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for L in paper_2601_07508_b200/libfpmm_b200.so abvar/libi8old.so; do
  for shape in "52 8192 8192 8192" "20 8192 8192 8192" "36 8192 8192 8192" "48 10923 32768 32" "50 1024 1024 1024"; do
    echo "$L $shape: $(FPMM_B200_LIB=$L ENGINE=i8 timeout 120 python tools/one_product.py $shape 5 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
  done
  FPMM_B200_LIB=$L timeout 300 python tools/bench_configs.py --only c1,unbalanced --engines auto --out gpurun_out/cfg_i8_$(basename $L .so)_$r.json > /dev/null 2>&1
done; done
