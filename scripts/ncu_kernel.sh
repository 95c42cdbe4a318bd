#!/bin/bash
# ncu --set full of one kernel of the bench step: NCU_K=<regex> [TAG=name] bash scripts/ncu_kernel.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:?}" -s ${NCU_S:-8} -c 1 \
    -o gpurun_out/${TAG:-kernel} -f python bench.py ${BENCH_ARGS:-} --steps 16 --warmup 3 --graph-steps 4 --sets 4 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/ncu_${TAG:-kernel}.log 2>&1; echo "ncu ${TAG:-kernel} rc=$?"
