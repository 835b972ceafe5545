# A/B of pack_b_rns (shared-memory transpose, FPMM_B200_RNS_PACKB_SMEM=1) vs pack_b_rns_direct (default)
for r in 1 2; do for f in 1 0; do
  for b in 20 36 52; do
    echo "smem=$f $b: $(FPMM_B200_RNS_PACKB_SMEM=$f ENGINE=rns timeout 120 python tools/one_product.py $b 8192 8192 8192 3 | tail -1 | grep -o "pack_ms.: [0-9.]*" | tr '\n' ' ')"
  done
done; done
timeout 600 python -m pytest tests/test_parity_rns_gpu.py tests/test_parity_gpu.py tests/test_dist_gpu.py -k "rns or None" -m gpu -x -q 2>&1 | tail -1
