# rns_kernel time vs K at m = n = 16384, 40-bit (per-pass overhead of short-K passes)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for S in 0 200; do for k in 256 512 1024 2048 4096; do
  echo "sleep=$S k=$k: $(FPMM_B200_RNS_EPI_SLEEP=$S ENGINE=rns timeout 120 python tools/one_product.py 40 16384 $k 16384 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*\|recon_ms.: [0-9.]*\|words.: [0-9]*" | tr '\n' ' ')"
done; done
