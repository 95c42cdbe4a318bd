#!/bin/bash
# Round-2 A/B on one GPU: build, GPU tests, multicast probe, bench step with / without the
# lookup's TSV_LOOKUP_INPUTS_READY (--no-extras: the default workload line only).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
if [[ -z "${NO_TESTS:-}" ]]; then
  timeout ${TEST_TIMEOUT:-1800} python -m pytest tests -m "gpu" -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -${PYTEST_TAIL:-6} gpurun_out/pytest_gpu.log
fi
if [[ -n "${PROBE:-}" ]]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_multicast scripts/probe_multicast.cu -lcuda && timeout 60 /tmp/probe_multicast > gpurun_out/probe_multicast.log 2>&1; echo "probe rc=$?"; cat gpurun_out/probe_multicast.log
fi
eval "set -- ${AB_ARGS:-'' '--no-lookup-ready'}"
n=0
for a in "$@"; do
  n=$((n+1))
  for rep in 1 2; do
    timeout 300 python bench.py --steps 1024 --warmup 32 --no-cpu-baseline --e2e-steps 0 --no-extras $a > gpurun_out/ab_$n.json 2>gpurun_out/ab_$n.err || tail -3 gpurun_out/ab_$n.err
    python -c "import json;d=json.load(open('gpurun_out/ab_$n.json'));r=d['roofline'];print('[$a]', round(d['ms_per_step']*1e3,2),'us/step p10/p90',round(d['ms_per_step_spread']['p10']*1e3,2),round(d['ms_per_step_spread']['p90']*1e3,2),'; race', round(r['launch_us'],2),'us frac',round(r['frac'],3), 'call', round(r.get('verify_call',{}).get('launch_us',0),2))"
  done
done
if [[ -n "${BREAKDOWN:-}" ]]; then
  timeout 300 python bench.py --steps 512 --warmup 32 --no-cpu-baseline --e2e-steps 0 --no-extras --breakdown > gpurun_out/breakdown.json 2>gpurun_out/breakdown.err; python -c "import json;d=json.load(open('gpurun_out/breakdown.json'));print('breakdown', d.get('breakdown'))"
fi
