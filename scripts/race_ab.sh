#!/bin/bash
# A/B of race-kernel compile-time variants on one GPU: for each flag set in AB_FLAGS, build, run the
# GPU verify/race parity tests (PARITY=0 skips them), then the bench step (no extras) REPS times.
# usage: AB_FLAGS="'' '-DX=1'" bash scripts/race_ab.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import oracle; oracle.build()" > gpurun_out/oracle_build.log 2>&1
eval "set -- ${AB_FLAGS:-''}"
n=0
for f in "$@"; do
  n=$((n+1))
  TSV_NVCC_EXTRA="$f" python -m paper_2406_14066_b200.build --force > gpurun_out/ab_build_$n.log 2>&1 || { echo "[$f] BUILD FAILED"; tail -5 gpurun_out/ab_build_$n.log; continue; }
  if [[ "${PARITY:-1}" == 1 ]]; then
    timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rng.py -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/ab_pytest_$n.log 2>&1; echo "[$f] parity rc=$? $(tail -1 gpurun_out/ab_pytest_$n.log)"
  fi
  for rep in $(seq 1 ${REPS:-2}); do
    timeout 300 python bench.py --steps ${STEPS:-1024} --warmup 32 --no-cpu-baseline --e2e-steps 0 --no-extras ${AB_BENCH:-} > gpurun_out/ab_$n.json 2>gpurun_out/ab_$n.err || tail -3 gpurun_out/ab_$n.err
    python -c "import json;d=json.load(open('gpurun_out/ab_$n.json'));r=d['roofline'];print('[$f]', round(d['ms_per_step']*1e3,2),'us/step; race', round(r['launch_us'],2),'us frac',round(r['frac'],3), 'call', round(r.get('verify_call',{}).get('launch_us',0),2))"
  done
done
