#!/bin/bash
# A/B of runtime env settings: AB_ENVS="'TSV_WEIGHTED=0' 'TSV_WEIGHTED=1'" bash scripts/ab_env.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
eval "set -- ${AB_ENVS:-''}"
n=0
for e in "$@"; do
  n=$((n+1))
  for rep in 1 2; do
    env $e timeout 300 python bench.py --steps 256 --warmup 16 --no-cpu-baseline --e2e-steps 0 ${AB_BENCH:-} > gpurun_out/abe_$n.json 2>gpurun_out/abe_$n.err || tail -3 gpurun_out/abe_$n.err
    python -c "import json;d=json.load(open('gpurun_out/abe_$n.json'));print('[$e]', round(d['ms_per_step']*1e3,2),'us/step; verify', round(d['roofline']['launch_us'],2),'us frac',round(d['roofline']['frac'],3), 'call', round(d['roofline'].get('verify_call',{}).get('launch_us',0),2))"
  done
done
