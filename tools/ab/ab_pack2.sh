# A/B: packers at their natural register count (abvar/lib8.so) vs capped at 64 registers (abvar/libnew.so)
for r in 1 2; do for L in abvar/lib8.so abvar/libnew.so; do
  for b in 20 36 52; do
    echo "$L $b: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py $b 8192 8192 8192 3 | tail -1 | grep -o "pack_ms.: [0-9.]*" | tr '\n' ' ')"
  done
done; done
