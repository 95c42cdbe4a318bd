#!/bin/bash
# Race-kernel waves sweep: for each build variant (SW_FLAGS), TSV_RACE_WAVES in SW_WAVES; prints the
# step time, the race kernel time / roofline fraction and the verify call.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
eval "set -- ${SW_FLAGS:-''}"
n=0
for f in "$@"; do
  n=$((n+1))
  TSV_NVCC_EXTRA="$f" python -m paper_2406_14066_b200.build --force > gpurun_out/sw_build_$n.log 2>&1 || { tail -5 gpurun_out/sw_build_$n.log; continue; }
  for w in ${SW_WAVES:-1 1.5 2 3}; do
    TSV_RACE_WAVES=$w timeout 300 python bench.py --steps 1024 --warmup 32 --no-cpu-baseline --e2e-steps 0 --no-extras ${SW_BENCH:-} > gpurun_out/sw_${n}_$w.json 2>gpurun_out/sw_${n}_$w.err || tail -3 gpurun_out/sw_${n}_$w.err
    python -c "import json;d=json.load(open('gpurun_out/sw_${n}_$w.json'));r=d['roofline'];print('[$f] waves $w:', round(d['ms_per_step']*1e3,2),'us/step; race', round(r['launch_us'],2),'us frac',round(r['frac'],3), 'call', round(r['verify_call']['launch_us'],2))"
  done
done
