# A/B of the RNS reconstruction: CRT fused into the last modulus pass (FPMM_B200_RNS_FUSED=1) vs rns_crt_kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for r in 1 2; do for f in 0 1; do
  echo "fused=$f: $(FPMM_B200_RNS_FUSED=$f timeout 300 python bench.py --no-e2e --no-cpu --no-engines --steps 5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])')"
done; done
