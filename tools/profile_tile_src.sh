#!/bin/bash
# source-level ncu capture of rns_tile_kernel at 16384 x 256 x 16384, 40 bits
cd "${GRAFT_REPO_ROOT:-/root/repo}"; out=gpurun_out; mkdir -p $out
shape=${SHAPE:-"40 16384 256 16384"}
FPMM_B200_RNS_TILE=1 ENGINE=rns timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"rns_tile" -c 1 -o $out/prof_src python tools/one_product.py $shape 1 > /dev/null 2>&1
ncu -i $out/prof_src.ncu-rep --page source --csv --print-source cuda > $out/prof_src.cuda.csv 2>&1
ncu -i $out/prof_src.ncu-rep --page source --csv --print-source sass > $out/prof_src.sass.csv 2>&1
gzip -f $out/prof_src.cuda.csv $out/prof_src.sass.csv
rm -f $out/prof_src.ncu-rep
ls -la $out
