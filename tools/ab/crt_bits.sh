# CRT kernel time per bitsize at 8192^3 (recon_ms), plus k = 256 (C5 class)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for b in 20 22 24 26 28 32 36 40 44 48 52; do
  echo "$b: $(ENGINE=rns timeout 120 python tools/one_product.py $b 8192 8192 8192 3 | tail -1 | grep -o "recon_ms.: [0-9.]*\|words.: [0-9]*" | tr '\n' ' ')"
done
echo "k=256: $(ENGINE=rns timeout 120 python tools/one_product.py 40 16384 256 16384 3 | tail -1 | grep -o "gemm_ms.: [0-9.]*\|recon_ms.: [0-9.]*" | tr '\n' ' ')"
