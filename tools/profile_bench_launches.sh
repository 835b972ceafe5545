#!/bin/bash
# ncu launch list of the default bench command with DRAM bytes per launch
# (serialised, cold-cache per launch: shares and traffic, not bench values),
# plus full captures of the current RNS kernels at 8192^3 / 52 bits.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; out=gpurun_out; mkdir -p $out
tag=${TAG:-r2}
FPMM_BENCH_DETAIL=$out/bench_detail_under_ncu.json timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches_bench_$tag.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-engines > $out/bench_under_ncu.log 2>&1
ENGINE=rns timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rns_kernel|rns_crt|pack_._rns" -c 4 \
    -o $out/prof_rns_b52_$tag python tools/one_product.py 52 8192 8192 8192 1 > /dev/null 2>&1
python tools/ncu_summary.py $out/prof_rns_b52_$tag.ncu-rep > $out/prof_rns_b52_$tag.json 2>/dev/null
ls -la $out | tail -5
