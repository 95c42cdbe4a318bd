#!/bin/bash
# compute-sanitizer over tests/sanitize_worker.py (every concurrency-heavy path, checked against the
# oracle): memcheck, racecheck, synccheck, initcheck, only libtsv's kernels instrumented.
# usage: bash scripts/sanitize.sh [paths...]      logs: gpurun_out/sanitizer/<tool>.log
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out/sanitizer
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sanitizer/build.log 2>&1 || { tail -20 gpurun_out/sanitizer/build.log; exit 1; }
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [[ $tool == racecheck ]] && extra="--racecheck-report all"
  [[ $tool == memcheck ]] && extra="--check-device-heap yes"
  t0=$(date +%s)
  filt="--kernel-name kns=tsv"
  [[ $tool == initcheck ]] && filt=""   # initcheck must see torch's writes too
  timeout 900 $CS --tool $tool $extra $filt --print-limit 50 --error-exitcode 99 \
      python tests/sanitize_worker.py "$@" > gpurun_out/sanitizer/$tool.log 2>&1
  rc=$?
  echo "$tool rc=$rc $(( $(date +%s) - t0 ))s: $(grep -c SANITIZE-OK gpurun_out/sanitizer/$tool.log) paths ok; $(grep 'ERROR SUMMARY' gpurun_out/sanitizer/$tool.log | tail -1)"
done
