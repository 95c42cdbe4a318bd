#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for rep in 1; do for f in "--breakdown" "--fused"; do
  timeout 300 python bench.py --steps 512 --warmup 16 --no-cpu-baseline --e2e-steps 0 $f > gpurun_out/f.json 2>gpurun_out/f.err || tail -3 gpurun_out/f.err
  python -c "import json;d=json.load(open('gpurun_out/f.json'));print('fused' if d['config']['fused'] else 'unfused', round(d['ms_per_step']*1e3,2),'us/step; verify', round(d['roofline']['launch_us'],2), d.get('breakdown_us_per_launch'))"
done; done
