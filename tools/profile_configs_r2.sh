#!/bin/bash
# ncu (speed of light, memory, tensor pipe) of one rns_kernel launch at C3 (first row block) and C4
cd "${GRAFT_REPO_ROOT:-/root/repo}"; out=gpurun_out; mkdir -p $out
for shape in "52 32768 32768 32768" "48 4096 262144 4096"; do
  set -- $shape; tag=b$1_k$3
  ENGINE=rns timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats \
    --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:"rns_kernel" -c 1 --csv --page raw python tools/one_product.py $shape 1 > $out/ncu_cfg_$tag.csv 2>/dev/null
done
ls -la $out
