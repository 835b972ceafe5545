# A/B of the RNS packers: digit form (dp4a) vs modulus pairs on the FP64 pipe (FPMM_B200_RNS_PACK_FP64=1)
for r in 1 2; do for f in 0 1; do
  for b in 20 36 52; do
    echo "fp64=$f $b: $(FPMM_B200_RNS_PACK_FP64=$f ENGINE=rns timeout 120 python tools/one_product.py $b 8192 8192 8192 3 | tail -1 | grep -o "pack_ms.: [0-9.]*\|gemm_ms.: [0-9.]*" | tr '\n' ' ')"
  done
done; done
FPMM_B200_RNS_PACK_FP64=1 timeout 600 python -m pytest tests/test_parity_rns_gpu.py tests/test_parity_gpu.py tests/test_dist_gpu.py -k "rns or None" -m gpu -x -q 2>&1 | tail -1
