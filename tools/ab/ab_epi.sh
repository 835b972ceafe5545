# A/B of the RNS epilogue width: 8 warps (default build) vs 16 (abvar/lib_epi16.so, FPMM_B200_RNS_EPI_WARPS=16)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
FPMM_B200_LIB=abvar/lib_epi16.so timeout 600 python -m pytest tests/test_parity_rns_gpu.py -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for L in paper_2601_07508_b200/libfpmm_b200.so abvar/lib_epi16.so; do
  for b in 20 36 52; do
    echo "$L $b: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py $b 8192 8192 8192 3 | tail -1 | grep -o "pack_ms.: [0-9.]*\|gemm_ms.: [0-9.]*\|recon_ms.: [0-9.]*" | tr '\n' ' ')"
  done
  echo "$L C5: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py 40 65536 256 65536 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*\|recon_ms.: [0-9.]*\|total_ms.: [0-9.]*" | tr '\n' ' ')"
  echo "$L C3: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py 52 32768 32768 32768 1 | tail -1 | grep -o "gemm_ms.: [0-9.]*\|recon_ms.: [0-9.]*\|total_ms.: [0-9.]*" | tr '\n' ' ')"
done; done
