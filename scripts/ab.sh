#!/bin/bash
# A/B libtsv variants (paper_2406_14066_b200/lib/exp/*.so) on the bench (no rebuild)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
for lib in paper_2406_14066_b200/lib/exp/*.so; do
  for c in ${CHUNKS:-2048}; do
    TSV_LIB_PATH=$PWD/$lib timeout 300 python bench.py --steps 256 --warmup 16 --no-cpu-baseline --e2e-steps 0 --chunk $c > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$(basename $lib)', $c, round(d['ms_per_step']*1e3,2),'us/step; verify', round(d['roofline']['launch_us'],2),'us')"
  done
done
