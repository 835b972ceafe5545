# A/B of the gathered row-chunk pipeline at world size 1 (bench --force-dist, NCCL path)
for c in 1 4 2; do
  FPMM_B200_DIST_CHUNKS=$c timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
    --master-addr 127.0.0.1 --master-port 2951$c bench.py --force-dist --no-cpu --no-e2e --steps 3 \
    > gpurun_out/bench_fd_c$c.json 2> gpurun_out/bench_fd_c$c.err
done
