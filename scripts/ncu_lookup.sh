#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
prof() {  # $1 tag
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$1.log 2>&1 || { tail -20 gpurun_out/build_$1.log; exit 1; }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:ngram_lookup -s 8 -c 1 \
      -o gpurun_out/lookup_$1 -f python bench.py --steps 16 --warmup 3 --graph-steps 4 --sets 4 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_$1.log 2>&1; echo "ncu $1 rc=$?"
}
prof new
cp scripts/lookup_old.cu.tmp paper_2406_14066_b200/csrc/lookup.cu
prof old
