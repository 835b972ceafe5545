# A/B of the CRT finalisation: one reduction (default) vs two (FPMM_B200_RNS_CRT_COMB=0)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_parity_rns_gpu.py tests/test_fullsize_gpu.py tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for C in 1 0; do
  for b in 20 28 36 44 52; do
    echo "comb=$C $b: $(FPMM_B200_RNS_CRT_COMB=$C ENGINE=rns timeout 120 python tools/one_product.py $b 8192 8192 8192 3 | tail -1 | grep -o "recon_ms.: [0-9.]*" | tr '\n' ' ')"
  done
  echo "comb=$C k=256: $(FPMM_B200_RNS_CRT_COMB=$C ENGINE=rns timeout 120 python tools/one_product.py 40 16384 256 16384 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*\|recon_ms.: [0-9.]*" | tr '\n' ' ')"
done; done
