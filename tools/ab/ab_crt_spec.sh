# A/B of the CRT kernel: specialised on (planes, groups) vs the generic one (FPMM_B200_RNS_CRT_SPEC=0)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_rns_gpu.py tests/test_fullsize_gpu.py -m gpu -x -q 2>&1 | tail -3
for r in 1 2; do for f in 0 1; do
  echo "spec=$f: $(FPMM_B200_RNS_CRT_SPEC=$f timeout 300 python bench.py --no-e2e --no-cpu --steps 5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], d["memory_side"])')"
done; done
for f in 0 1; do
  FPMM_B200_RNS_CRT_SPEC=$f timeout 600 python tools/bench_configs.py --only c3,c5 --engines rns --out gpurun_out/cfg_spec$f.json > /dev/null 2>&1
  echo "spec=$f"; python -c "
import json; [print(r['m'],r['k'],r['n'],r['bits'],r['ms'],r['eff_gflops']) for r in json.load(open('gpurun_out/cfg_spec$f.json'))]"
done
ENGINE=rns timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rns_crt" -c 1 -o gpurun_out/prof_crt_spec python tools/one_product.py 52 8192 8192 8192 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_crt_spec.ncu-rep > gpurun_out/prof_crt_spec.json 2>/dev/null
