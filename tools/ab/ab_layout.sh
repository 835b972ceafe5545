#!/bin/bash
# RNS packed layout [block][k-block][modulus] (in-tree) vs [block][modulus][k-block] (abvar/liblayoutold.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests/test_parity_rns_gpu.py tests/test_fullsize_gpu.py tests/test_dist_gpu.py -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for L in paper_2601_07508_b200/libfpmm_b200.so abvar/liblayoutold.so; do
  for shape in "52 8192 8192 8192" "20 8192 8192 8192" "48 4096 262144 4096"; do
    echo "$L $shape: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py $shape 3 | tail -1 | grep -o "pack_ms.: [0-9.]*\|gemm_ms.: [0-9.]*\|recon_ms.: [0-9.]*" | tr '\n' ' ')"
  done
  FPMM_B200_LIB=$L timeout 300 python tools/bench_configs.py --only c3,c4,c5 --engines rns --out gpurun_out/lay_$(basename $L .so)_$r.json > /dev/null 2>&1
  python -c "
import json
for x in json.load(open('gpurun_out/lay_$(basename $L .so)_$r.json')): print('$L', x['m'], x['k'], x['n'], x['ms'], x['eff_gflops'], x['pack_ms'])"
done; done
