#!/bin/bash
# Round-2 check on one GPU: build, GPU tests, sanitizer logs, the default bench line (with every
# workload sub-object) and the N = 2 bench path with both ranks on the one GPU.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout ${TEST_TIMEOUT:-1800} python -m pytest tests -m "gpu" -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -${PYTEST_TAIL:-15} gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
if [[ -n "${SAN:-}" ]]; then bash scripts/sanitize.sh; fi
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [[ -n "${SHARED2:-}" ]]; then
  TSV_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29517 bench.py --gpus 2 --steps 64 --warmup 3 --e2e-steps 2 > gpurun_out/shared2.json 2> gpurun_out/shared2.err
  echo "shared2 rc=$?"; head -c 600 gpurun_out/shared2.json; tail -3 gpurun_out/shared2.err
fi
