# A/B of the RNS epilogue: two warp groups on alternate passes (default) vs all 16 warps on every pass (FPMM_B200_RNS_PINGPONG=0)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_parity_rns_gpu.py tests/test_fullsize_gpu.py tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for PP in 1 0; do
  for b in 20 36 52; do
    echo "pp=$PP $b: $(FPMM_B200_RNS_PINGPONG=$PP ENGINE=rns timeout 120 python tools/one_product.py $b 8192 8192 8192 3 | tail -1 | grep -o "pack_ms.: [0-9.]*\|gemm_ms.: [0-9.]*\|recon_ms.: [0-9.]*" | tr '\n' ' ')"
  done
  for k in 256 1024; do
  echo "pp=$PP k=$k: $(FPMM_B200_RNS_PINGPONG=$PP ENGINE=rns timeout 120 python tools/one_product.py 40 16384 $k 16384 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*\|recon_ms.: [0-9.]*" | tr '\n' ' ')"
  done
  echo "pp=$PP C5: $(FPMM_B200_RNS_PINGPONG=$PP ENGINE=rns timeout 120 python tools/one_product.py 40 65536 256 65536 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*\|total_ms.: [0-9.]*" | tr '\n' ' ')"
done; done
