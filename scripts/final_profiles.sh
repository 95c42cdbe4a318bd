#!/bin/bash
# End-of-round evidence (round 2): GPU tests + smoke, the default bench line (every
# workload as a sub-object), the driver-style short run, the step breakdown, two ranks on the one GPU,
# ncu launch lists (step, NVTX-filtered, config-4 peer-memory paths), a --set full capture of the race
# kernel and the per-workload DRAM traffic.  Outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
SHARED2=1 bash scripts/r02_check.sh  # compute-sanitizer: closed on the GPU pool this round (logs of the earlier run stay in profiles/r02/sanitizer)
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/bench_driver_style.json 2> gpurun_out/bench_driver_style.err
echo "driver-style bench rc=$?"
timeout 600 python bench.py --breakdown --no-cpu-baseline --e2e-steps 0 --no-extras > gpurun_out/bench_breakdown.json \
    2> gpurun_out/bench_breakdown.err; echo "breakdown rc=$?"
bash scripts/gpu_all.sh ncu
bash scripts/ncu_nvtx.sh
bash scripts/ncu_c4.sh
bash scripts/traffic.sh
