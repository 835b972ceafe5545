#!/bin/bash
# ncu evidence for the RNS / int8 engines (run under gpurun, one GPU):
#   full captures of the product kernels at 8192^3 and the bench's launch list.
set -x
out=gpurun_out
ENGINE=rns timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rns_kernel|rns_crt|pack_._rns" -c 4 \
    -o $out/prof_rns_b52 python tools/one_product.py 52 8192 8192 8192 1 > $out/ncu_rns_b52.log 2>&1
ENGINE=rns timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rns_kernel|rns_crt" -c 2 \
    -o $out/prof_rns_b20 python tools/one_product.py 20 8192 8192 8192 1 > $out/ncu_rns_b20.log 2>&1
ENGINE=i8 timeout 900 ncu --set full --clock-control none -k regex:"mwi8_kernel" -c 1 \
    -o $out/prof_i8_b52 python tools/one_product.py 52 8192 8192 8192 1 > $out/ncu_i8_b52.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $out/bench_under_ncu.log 2>&1
ls -la $out
