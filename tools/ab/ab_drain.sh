# A/B of the RNS epilogue order: drain all columns then release (default) vs release after the last load (abvar/lib_drain0.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests/test_parity_rns_gpu.py tests/test_fullsize_gpu.py -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for L in paper_2601_07508_b200/libfpmm_b200.so abvar/lib_drain0.so; do
  for b in 20 36 52; do
    echo "$L $b: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py $b 8192 8192 8192 3 | tail -1 | grep -o "pack_ms.: [0-9.]*\|gemm_ms.: [0-9.]*\|recon_ms.: [0-9.]*" | tr '\n' ' ')"
  done
  echo "$L C5: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py 40 65536 256 65536 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*\|total_ms.: [0-9.]*" | tr '\n' ' ')"
  echo "$L C5-16k: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py 40 16384 256 16384 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*\|recon_ms.: [0-9.]*\|total_ms.: [0-9.]*" | tr '\n' ' ')"
done; done
