# where the time of a short-K rns_kernel goes (FPMM_B200_RNS_DEBUG: 1 no stores, 2 no epilogue work, 4 no MMAs, 6 neither)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for D in 0 1 2 4 6 0; do for k in 256 1024; do
  echo "debug=$D k=$k: $(FPMM_B200_RNS_DEBUG=$D ENGINE=rns timeout 120 python tools/one_product.py 40 16384 $k 16384 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*" | tr '\n' ' ')"
done; done
