#!/bin/bash
# pack_a_rns on a 2-D grid (in-tree) vs the 1-D grid-stride form with 64-bit div/mod per item (abvar/libpackaold.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for L in paper_2601_07508_b200/libfpmm_b200.so abvar/libpackaold.so; do
  for shape in "52 8192 8192 8192" "20 8192 8192 8192" "48 4096 262144 4096" "40 65536 256 65536"; do
    echo "$L $shape: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py $shape 3 | tail -1 | grep -o "pack_ms.: [0-9.]*")"
  done
done; done
