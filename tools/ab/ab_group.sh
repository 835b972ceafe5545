# RNS rasterisation group size sweep (pair-tile rows per group) with the flat pass order
for r in 1 2; do for gsz in 16 8 32 4 12; do
  for b in 20 52; do
    echo "group=$gsz $b: $(FPMM_B200_RNS_GROUP=$gsz ENGINE=rns timeout 120 python tools/one_product.py $b 8192 8192 8192 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*")"
  done
done; done
for gsz in 16 8 32; do
  FPMM_B200_RNS_GROUP=$gsz ENGINE=rns timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:rns_kernel -c 1 python tools/one_product.py 52 8192 8192 8192 1 2>&1 | grep -E "dram__bytes|duration" | sed "s/^/group=$gsz /"
done
