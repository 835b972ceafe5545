# A/B of the RNS pass order: FPMM_B200_RNS_FLAT=0 (modulus-major per pair) vs 1 (one flat sequence)
for r in 1 2; do for f in 0 1; do
  for b in 20 36 52; do
    echo "flat=$f $b: $(FPMM_B200_RNS_FLAT=$f ENGINE=rns timeout 120 python tools/one_product.py $b 8192 8192 8192 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
  done
done; done
for f in 0 1; do
  FPMM_B200_RNS_FLAT=$f ENGINE=rns timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:rns_kernel -c 1 python tools/one_product.py 52 8192 8192 8192 1 2>&1 | grep -E "dram__bytes|duration|hit_rate" | sed "s/^/flat=$f /"
done
FPMM_B200_RNS_FLAT=1 timeout 600 python -m pytest tests/test_parity_rns_gpu.py -m gpu -x -q 2>&1 | tail -1
