#!/bin/bash
# Sweep a compile-time macro of the recon kernel: tools/macro_sweep.sh MACRO "v1 v2 ..." [env VAR=val ...]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
macro=$1; vals=$2; shift 2
for v in $vals; do
  touch paper_2308_02494_b200/csrc/recon_tc16.cu
  make EXTRA=-D$macro=$v >/dev/null 2>&1 || { echo "build failed $macro=$v"; exit 1; }
  echo -n "$macro=$v: "; env "$@" tools/bench_ab.sh APMG_NONE "x" --no-e2e
done
touch paper_2308_02494_b200/csrc/recon_tc16.cu
make >/dev/null 2>&1
