#!/bin/bash
# A/B of compile-time variants: AB_FLAGS="'' '-DX=0'" bash scripts/ab_build.sh  (bench step + verify per launch)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
eval "set -- ${AB_FLAGS:-''}"
n=0
for f in "$@"; do
  n=$((n+1))
  TSV_NVCC_EXTRA="$f" python -m paper_2406_14066_b200.build --force > gpurun_out/ab_build_$n.log 2>&1 || { tail -5 gpurun_out/ab_build_$n.log; continue; }
  for rep in 1 2; do
    timeout 300 python bench.py --steps 256 --warmup 16 --no-cpu-baseline --e2e-steps 0 ${AB_BENCH:-} > gpurun_out/ab_$n.json 2>gpurun_out/ab_$n.err || tail -3 gpurun_out/ab_$n.err
    python -c "import json;d=json.load(open('gpurun_out/ab_$n.json'));print('[$f]', round(d['ms_per_step']*1e3,2),'us/step; verify', round(d['roofline']['launch_us'],2),'us frac',round(d['roofline']['frac'],3), 'call', round(d['roofline'].get('verify_call',{}).get('launch_us',0),2))"
  done
done
