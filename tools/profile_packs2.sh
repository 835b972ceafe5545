#!/bin/bash
# stall reasons and memory chart of the RNS packers at 8192^2, 52 bits
cd "${GRAFT_REPO_ROOT:-/root/repo}"; out=gpurun_out; mkdir -p $out
ENGINE=rns timeout 600 ncu --set full --clock-control none -k regex:"pack_._rns" -c 2 \
  -o $out/prof_pack2 python tools/one_product.py 52 8192 8192 8192 1 > /dev/null 2>&1
ncu -i $out/prof_pack2.ncu-rep --page details --csv > $out/prof_pack2.details.csv 2>/dev/null
ncu -i $out/prof_pack2.ncu-rep --page raw --csv > $out/prof_pack2.raw.csv 2>/dev/null
gzip -f $out/prof_pack2.raw.csv; rm -f $out/prof_pack2.ncu-rep
