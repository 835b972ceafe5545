#!/bin/bash
# one gpurun call: GPU tests, then a default bench run (logs under gpurun_out/)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest.log
if [ -z "$NO_BENCH" ]; then
  FPMM_BENCH_DETAIL=gpurun_out/bench_detail.json timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2> gpurun_out/bench.err
  echo "bench rc=$?" >> gpurun_out/bench.err
fi
tail -3 gpurun_out/pytest.log; tail -c 3000 gpurun_out/bench.log
