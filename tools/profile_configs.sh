#!/bin/bash
# Per-config RNS timing (bench_configs) and an ncu launch list with DRAM bytes
# per launch for one product of C3, C4 and C5 (serialised, cold-cache:
# shares and traffic, not bench values).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; out=gpurun_out; mkdir -p $out
tag=${TAG:-r2}
timeout 900 python tools/bench_configs.py --only c3,c4,c5 --engines rns --out $out/configs_$tag.json > $out/configs_$tag.log 2>&1
for c in "52 32768 32768 32768" "48 4096 262144 4096" "40 65536 256 65536"; do
  set -- $c
  ENGINE=rns timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv \
      --log-file $out/launches_${2}_${tag}.csv python tools/one_product.py $1 $2 $3 $4 1 > $out/one_${2}_${tag}.log 2>&1
done
ls -la $out | tail -8
