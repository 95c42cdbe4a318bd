#!/bin/bash
# quick GPU iteration: build, verify parity subset, bench verify timing, chunk sweep
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -${PYTEST_TAIL:-4} gpurun_out/pytest_gpu.log
for c in ${CHUNKS:-1024 2048 4096}; do
  timeout 300 python bench.py --steps 256 --warmup 16 --no-cpu-baseline --e2e-steps 0 --chunk $c > gpurun_out/sweep_$c.json 2>gpurun_out/sweep_$c.err || tail -5 gpurun_out/sweep_$c.err
  python -c "import json;d=json.load(open('gpurun_out/sweep_$c.json'));print($c, round(d['ms_per_step']*1e3,2),'us/step; verify', round(d['roofline']['launch_us'],2),'us frac',round(d['roofline']['frac'],3))"
done
if [[ -n "${NCU:-}" ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"verify|lookup|goodput|update" -c 300 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 32 --warmup 3 --graph-steps 8 --sets 4 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_bench.log 2>&1; echo "ncu-launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-verify_race}" -s ${NCU_S:-8} -c ${NCU_C:-1} \
      -o gpurun_out/verify_full -f python bench.py --steps 16 --warmup 3 --graph-steps 4 --sets 4 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
fi
