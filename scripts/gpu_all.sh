#!/bin/bash
# One gpurun call: build, GPU parity tests, smoke, a bench line, ncu launch list + full capture.
# usage: bash scripts/gpu_all.sh [tests|bench|ncu|all] ...
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
what="${1:-all}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
if [[ "$what" == tests || "$what" == all ]]; then
  timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -25 gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
fi
if [[ "$what" == bench || "$what" == all ]]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
fi
if [[ "$what" == ncu || "$what" == all ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"verify|lookup|goodput|update" -c 400 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 64 --warmup 3 --graph-steps 8 --sets 4 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_bench.log 2>&1; echo "ncu-launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:verify_race -s 8 -c 2 \
      -o gpurun_out/verify_full -f python bench.py --steps 16 --warmup 3 --graph-steps 4 --sets 4 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
  tail -3 gpurun_out/ncu_full.log
fi
