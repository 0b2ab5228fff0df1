#!/bin/bash
# Sweep the warp-aggregation round cap of the scatter (compile-time APMG_AGG_ROUNDS).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for r in ${1:-1 2 3 4}; do
  touch paper_2308_02494_b200/csrc/recon_tc16.cu
  make EXTRA=-DAPMG_AGG_ROUNDS=$r >/dev/null 2>&1 || { echo "build failed r=$r"; exit 1; }
  echo -n "rounds=$r: "; tools/bench_ab.sh APMG_NONE "x" --no-e2e
done
touch paper_2308_02494_b200/csrc/recon_tc16.cu
make >/dev/null 2>&1
