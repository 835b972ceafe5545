#!/bin/bash
# ncu of the RNS packers at C4 (4096 x 262144 x 4096, 48 bits) and 8192^3 52 bits
cd "${GRAFT_REPO_ROOT:-/root/repo}"; out=gpurun_out; mkdir -p $out
for shape in "48 4096 262144 4096" "52 8192 8192 8192"; do
  set -- $shape; tag=b$1_k$3
  ENGINE=rns timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pack_._rns" -c 2 \
    -o $out/prof_pack_$tag python tools/one_product.py $shape 1 > /dev/null 2>&1
  ncu -i $out/prof_pack_$tag.ncu-rep --page details --csv > $out/prof_pack_$tag.details.csv 2>/dev/null
  ncu -i $out/prof_pack_$tag.ncu-rep --page source --csv --print-source sass > $out/prof_pack_$tag.sass.csv 2>/dev/null
  gzip -f $out/prof_pack_$tag.sass.csv; rm -f $out/prof_pack_$tag.ncu-rep
done
ls -la $out
