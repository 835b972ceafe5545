#!/bin/bash
# C4 DRAM with and without pacing; C3 pacing x rasterisation group
cd "${GRAFT_REPO_ROOT:-/root/repo}"; out=gpurun_out; mkdir -p $out
for pace in 0 64; do
  FPMM_B200_RNS_PACE=$pace ENGINE=rns timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none --csv -k regex:rns_kernel -c 1 \
      --log-file $out/launches_c4_pace$pace.csv python tools/one_product.py 48 4096 262144 4096 1 > /dev/null 2>&1
  grep rns_kernel $out/launches_c4_pace$pace.csv | awk -F'","' -v p=$pace '{print "c4 pace", p, $13, $15}'
done > $out/ab_pace2.txt
for grp in 4 8 32; do
  for pace in 0 64; do
    echo "group=$grp pace=$pace $(FPMM_B200_RNS_GROUP=$grp FPMM_B200_RNS_PACE=$pace timeout 600 python tools/bench_configs.py --only c3,c4 --engines rns 2>&1 | grep -o '"ms": [0-9.]*' | tr '\n' ' ')"
  done
done >> $out/ab_pace2.txt 2>&1
cat $out/ab_pace2.txt
