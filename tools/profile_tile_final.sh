#!/bin/bash
# ncu --set full of the default short-K path (rns_tile_kernel, 16384 x 256 x 16384, 40 bits), summarised on the box
cd "${GRAFT_REPO_ROOT:-/root/repo}"; out=gpurun_out; mkdir -p $out
ENGINE=rns timeout 600 ncu --set full --clock-control none -k regex:"rns_tile|pack_._rns" -c 3 \
  -o $out/prof_tile_final python tools/one_product.py 40 16384 256 16384 1 > /dev/null 2>&1
python tools/ncu_summary.py $out/prof_tile_final.ncu-rep tile_final > $out/ncu_tile_16384_k256_b40.json 2>/dev/null
rm -f $out/prof_tile_final.ncu-rep
