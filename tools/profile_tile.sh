#!/bin/bash
# ncu --set full of rns_tile_kernel (on-chip CRT) and rns_kernel on the short-K
# (C5 class) and 8192^3 shapes: what bounds each.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; out=gpurun_out; mkdir -p $out
for shape in "40 16384 256 16384" "20 8192 8192 8192"; do
  set -- $shape; tag=b$1_k$3
  for tile in 1 0; do
    FPMM_B200_RNS_TILE=$tile ENGINE=rns timeout 600 ncu --set full --clock-control none --import-source on \
      -k regex:"rns_tile|rns_kernel|rns_crt" -c 2 -o $out/prof_tile${tile}_$tag python tools/one_product.py $shape 1 > /dev/null 2>&1
  done
done
ls -la $out
for r in $out/prof_tile*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  gzip -f $b.raw.csv
done
[ -n "$KEEP_REP" ] || rm -f $out/prof_tile*.ncu-rep
ls -la $out
