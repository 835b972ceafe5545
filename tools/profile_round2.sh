#!/bin/bash
# Round-2 ncu evidence (one GPU): full captures of the RNS kernels at 8192^3
# (52 and 20 bits), the launch list of the default bench command, and the
# per-kernel times of C5 (65536 x 256 x 65536, 40 bits).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; out=gpurun_out; mkdir -p $out
tag=${TAG:-r2}
ENGINE=rns timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rns_kernel|rns_crt|pack_._rns" -c 4 \
    -o $out/prof_rns_b52_$tag python tools/one_product.py 52 8192 8192 8192 1 > $out/ncu_rns_b52.log 2>&1
ENGINE=rns timeout 900 ncu --set full --clock-control none -k regex:"rns_kernel|rns_crt" -c 2 \
    -o $out/prof_rns_b20_$tag python tools/one_product.py 20 8192 8192 8192 1 > $out/ncu_rns_b20.log 2>&1
ENGINE=rns timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches_c5_$tag.csv python tools/one_product.py 40 65536 256 65536 2 > $out/ncu_c5.log 2>&1
[ -z "$NO_LAUNCHES" ] && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_bench_$tag.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-engines > $out/bench_under_ncu.log 2>&1
for f in $out/prof_*_$tag.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.json 2>/dev/null; done
ls -la $out
