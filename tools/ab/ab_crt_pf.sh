# A/B of the CRT residue prefetch (default build) vs none (abvar/lib_nopf.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests/test_parity_rns_gpu.py -m gpu -x -q 2>&1 | tail -1
for L in paper_2601_07508_b200/libfpmm_b200.so abvar/lib_nopf.so; do
for b in 20 26 36 44 52; do
  echo "$L $b: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py $b 8192 8192 8192 3 | tail -1 | grep -o "recon_ms.: [0-9.]*" | tr '\n' ' ')"
done
echo "$L k=256: $(FPMM_B200_LIB=$L ENGINE=rns timeout 120 python tools/one_product.py 40 16384 256 16384 3 | tail -1 | grep -o "recon_ms.: [0-9.]*" | tr '\n' ' ')"
done
