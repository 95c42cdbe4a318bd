#!/bin/bash
# The N > 1 host path of bench.py on a one-GPU box: 2 ranks on cuda:0 over gloo (TSV_BENCH_SHARED_GPU=1).
# Checks the multi-rank plumbing (rank-0-only JSON line, max/sum over ranks, barriers); not a measurement.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
for wl in step greedy; do
  TSV_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29517 bench.py --gpus 2 --steps 64 --warmup 3 --e2e-steps 2 --workload $wl \
      > gpurun_out/shared2_$wl.json 2> gpurun_out/shared2_$wl.err; echo "shared-gpu 2 ranks $wl rc=$? lines=$(wc -l < gpurun_out/shared2_$wl.json)"
  head -c 400 gpurun_out/shared2_$wl.json; echo
done
