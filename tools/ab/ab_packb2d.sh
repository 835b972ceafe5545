#!/bin/bash
# pack_b_rns_direct on a 2-D grid without per-item 64-bit division (in-tree) vs the 1-D grid-stride form (abvar/libpackbold.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests/test_parity_rns_gpu.py tests/test_dist_gpu.py tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for L in paper_2601_07508_b200/libfpmm_b200.so abvar/libpackbold.so; do
  for shape in "52 8192 8192 8192" "20 8192 8192 8192" "48 4096 262144 4096" "40 65536 256 65536"; do
    echo "$L $shape: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py $shape 3 | tail -1 | grep -o "pack_ms.: [0-9.]*")"
  done
done; done
