# A/B of the fused CRT on the BASELINE configs (RNS engine)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for f in 0 1; do
  FPMM_B200_RNS_FUSED=$f timeout 600 python tools/bench_configs.py --only c1,c3,c4,c5 --engines rns --out gpurun_out/cfg_fused$f.json > /dev/null 2>&1
  echo "fused=$f"; python -c "
import json; [print(r['m'],r['k'],r['n'],r['bits'],r['ms'],r['eff_gflops']) for r in json.load(open('gpurun_out/cfg_fused$f.json'))]"
done
