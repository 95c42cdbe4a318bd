#!/bin/bash
# NVTX-filtered ncu launch list (tracing): only kernels launched inside the bench's
# "timed" range, attributed to the libtsv entry point (TSV_NVTX=1) that enqueued them at graph capture.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
timeout 600 ncu --nvtx --nvtx-include "bench:step/timed/" -k regex:"verify|lookup|goodput|update" --metrics gpu__time_duration.sum \
    --clock-control none -c ${NCU_C:-40} --csv --log-file gpurun_out/launches_nvtx.csv \
    python bench.py --nvtx --steps 16 --warmup 3 --graph-steps 4 --no-extras --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/ncu_nvtx.log 2>&1; echo "ncu nvtx rc=$?"; tail -3 gpurun_out/ncu_nvtx.log
