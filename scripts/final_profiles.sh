#!/bin/bash
# End-of-round evidence: GPU tests + smoke, the default bench line, every workload line, the ncu launch
# list of the default step and a --set full capture of the race kernel.  Outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
bash scripts/gpu_all.sh all
for wl in greedy logits config5; do
  timeout 600 python bench.py --workload $wl > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; echo "bench $wl rc=$?"
done
for m in none lazy dense p2p; do
  timeout 600 python bench.py --workload config4 --shard-mode $m > gpurun_out/bench_config4_$m.json 2> gpurun_out/bench_config4_$m.err; echo "bench config4 $m rc=$?"
done
BENCH_ARGS="--breakdown --no-cpu-baseline --e2e-steps 0" timeout 600 python bench.py --breakdown --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_breakdown.json 2> gpurun_out/bench_breakdown.err; echo "breakdown rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"verify|logit|softmax" -c 40 --csv \
    --log-file gpurun_out/launches_logits.csv python bench.py --workload logits --steps 8 --warmup 3 --graph-steps 4 > /dev/null 2>&1; echo "ncu logits rc=$?"
