#!/bin/bash
# Sweep how the tc16 scatter is split between the encode and the tensor-core waits.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for cfg in "$@"; do
  set -- $cfg
  touch paper_2308_02494_b200/csrc/recon_tc16.cu
  make EXTRA="-DTC16_SQ_I=$1 -DTC16_SQ_C=$2 -DTC16_SQ_E=$3" >/dev/null 2>&1 || { echo "build failed $cfg"; exit 1; }
  echo -n "sq=$cfg: "; tools/bench_ab.sh APMG_NONE "x" --no-e2e
done
touch paper_2308_02494_b200/csrc/recon_tc16.cu
make >/dev/null 2>&1
