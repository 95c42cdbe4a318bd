#!/bin/bash
# ncu launch lists of the config-4 vocab-sharded paths at N = 1 (per-kernel serialized times).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for m in ${C4_MODES:-p2p p2p_fused}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"verify|p2p" -c 40 --csv \
      --log-file gpurun_out/launches_c4_$m.csv python bench.py --workload config4 --shard-mode $m --steps 8 --warmup 3 \
      --graph-steps 4 --no-extras > /dev/null 2>&1; echo "ncu $m rc=$?"
done
