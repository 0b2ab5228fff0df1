#!/bin/bash
# A/B of ab/<name> builds or VAR=value switches against the default (ROUNDS rounds), after a smoke.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
ROUNDS=${ROUNDS:-3} bash tools/ab_bench.sh "$@" > /dev/null 2>&1
cat gpurun_out/ab.log
