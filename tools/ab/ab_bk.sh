# A/B of the RNS stage depth in k: abvar/lib8.so (kBK = 64) vs abvar/libnew.so (FPMM_B200_RNS_BK=128)
for r in 1 2; do for L in abvar/lib8.so abvar/libnew.so abvar/lib256.so; do
  for b in 20 36 52; do
    echo "$L $b: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py $b 8192 8192 8192 3 | tail -1 | grep -o "pack_ms.: [0-9.]*\|gemm_ms.: [0-9.]*\|recon_ms.: [0-9.]*" | tr '\n' ' ')"
  done
  echo "$L C5: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py 40 65536 256 65536 2 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
done; done
for L in abvar/libnew.so abvar/lib256.so; do FPMM_B200_LIB=$L timeout 600 python -m pytest tests/test_parity_rns_gpu.py tests/test_parity_gpu.py tests/test_dist_gpu.py -k "rns or None" -m gpu -x -q 2>&1 | tail -1; done
