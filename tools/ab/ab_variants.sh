for r in 1 2; do for L in abvar/lib8.so abvar/libnew.so; do
  echo "$L C5: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py 40 65536 256 65536 2 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
  ENGINE=rns bash tools/ab.sh 52 "$L" 1
  ENGINE=rns bash tools/ab.sh 20 "$L" 1
done; done
timeout 600 python -m pytest tests/test_parity_rns_gpu.py tests/test_parity_gpu.py tests/test_dist_gpu.py -k "rns or None" -m gpu -x -q 2>&1 | tail -2
