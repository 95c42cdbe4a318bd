#!/bin/bash
# For a box with >= 2 GPUs (not available in round 1): the multi-GPU paths end to end.
#  - GPU tests (the two-process peer-memory test then maps a real NVLink peer)
#  - the default step, request-sharded weak scaling, N = 2, 4, 8
#  - config 4 vocab-sharded: NCCL lazy two rounds vs the peer-memory (LL) exchange vs the race-epilogue
#    push (P2P_FUSED), N = 2, 4, 8; the strong-scaling step
#  - the multicast (NVLS) probe
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
NG=$(nvidia-smi -L | wc -l)
for n in 2 4 8; do
  [[ $n -le $NG ]] || continue
  run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --gpus $n "$@"; }
  run > gpurun_out/scale_step_$n.json 2> gpurun_out/scale_step_$n.err; echo "step N=$n rc=$?"
  run --workload strong > gpurun_out/scale_strong_$n.json 2> gpurun_out/scale_strong_$n.err; echo "strong N=$n rc=$?"
  for m in lazy p2p p2p_fused; do
    run --workload config4 --shard-mode $m > gpurun_out/scale_c4_${m}_$n.json 2> gpurun_out/scale_c4_${m}_$n.err; echo "config4 $m N=$n rc=$?"
  done
  # the lazy mode's key all-reduce is ncclAllReduce(max, uint64): NCCL's algorithm choice (NVLS = in-switch
  # reduction) is in its INFO log
  NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,COLL,TUNING run --workload config4 --shard-mode lazy --steps 8 --warmup 3 \
      > /dev/null 2> gpurun_out/nccl_c4_lazy_$n.log; echo "config4 lazy NCCL log N=$n rc=$? NVLS lines: $(grep -ci nvls gpurun_out/nccl_c4_lazy_$n.log)"
done
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_multicast scripts/probe_multicast.cu -lcuda && \
  timeout 60 /tmp/probe_multicast > gpurun_out/probe_multicast.log 2>&1; tail -3 gpurun_out/probe_multicast.log
