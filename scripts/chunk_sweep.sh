#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for c in ${CHUNKS:-1024 2048 4096 8192 16384}; do
  timeout 300 python bench.py --steps 256 --warmup 16 --no-cpu-baseline --e2e-steps 0 --chunk $c > gpurun_out/sweep_$c.json 2>gpurun_out/sweep_$c.err
  python -c "import json;d=json.load(open('gpurun_out/sweep_$c.json'));print($c, round(d['ms_per_step']*1e3,2),'us/step verify', round(d['roofline']['launch_us'],2),'us frac',round(d['roofline']['frac'],3))"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify_race -s 8 -c 1 \
   -o gpurun_out/verify_full -f python bench.py --steps 16 --warmup 3 --graph-steps 4 --sets 4 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
