#!/bin/bash
# A/B of the RNS producer pacing (FPMM_B200_RNS_PACE = k-blocks of lead over the
# slowest pair): long-K configs C3 / C4, the 8192^3 sweep, and DRAM bytes of C3.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; out=gpurun_out; mkdir -p $out
for pace in ${PACES:-0 32 64 128}; do
  echo "pace=$pace"
  FPMM_B200_RNS_PACE=$pace timeout 600 python tools/bench_configs.py --only ${CFGS:-c3,c4} --engines rns 2>&1 | grep -o '"m".*"eff_gflops": [0-9.]*'
done > $out/ab_pace.txt 2>&1
for pace in 0 ${NCU_PACE:-64}; do
  FPMM_B200_RNS_PACE=$pace ENGINE=rns timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none --csv -k regex:rns_kernel -c 1 \
      --log-file $out/launches_c3_pace$pace.csv python tools/one_product.py 52 32768 32768 32768 1 > /dev/null 2>&1
done
for pace in 0 ${SWEEP_PACE:-64}; do
  echo "sweep pace=$pace: $(FPMM_B200_RNS_PACE=$pace timeout 600 python bench.py --no-e2e --no-cpu --no-engines --steps 5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])')"
done >> $out/ab_pace.txt
cat $out/ab_pace.txt
for sl in ${SLICES:-64 128}; do
  echo "slice_kb=$sl"
  FPMM_B200_RNS_SLICE_KB=$sl timeout 600 python tools/bench_configs.py --only ${CFGS:-c3,c4} --engines rns 2>&1 | grep -o '"m".*"eff_gflops": [0-9.]*'
done >> $out/ab_pace.txt 2>&1
tail -6 $out/ab_pace.txt
