#!/bin/bash
# DRAM traffic per call of every bench workload (roofline "traffic"): ncu with cold caches
# (--cache-control all) over a short run of each workload; scripts/traffic_summary.py sums the
# kernels of one call -> gpurun_out/traffic.json, committed as profiles/r02/traffic.json (the capture bench.py reads).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for w in ${TRAFFIC_WORKLOADS:-step greedy logits config4 config5}; do
  timeout 600 ncu --metrics $M --cache-control all --clock-control none -k regex:"tsv|verify|lookup|goodput|update|logit|greedy|clear" \
      -c ${NCU_C:-120} --csv --log-file gpurun_out/traffic_$w.csv \
      python bench.py --workload $w --steps 8 --warmup 3 --graph-steps 4 --no-extras --no-cpu-baseline --e2e-steps 0 \
      > gpurun_out/traffic_$w.log 2>&1; echo "ncu $w rc=$?"
done
python scripts/traffic_summary.py gpurun_out gpurun_out/traffic.json  # committed as profiles/r02/traffic.json
