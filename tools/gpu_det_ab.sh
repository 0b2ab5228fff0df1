#!/bin/bash
# Deterministic-mode A/B: the default build against ab/<name> builds (args), two rounds, then the
# determinism tests.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for r in 1 2; do for v in default "$@"; do
lib=""; [ "$v" != default ] && lib="$PWD/ab/$v/libapmg_cuda.so"
APMG_DETERMINISTIC=1 APMG_LIB="$lib" timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-inference --no-render --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('DET $v', round(d['value']/1e6,1), round(d['roofline']['ms_per_launch'],4), d['final_l_rec'])"
done; done
timeout 600 python -m pytest tests -m gpu -q -x -k "determin or multirank" 2>&1 | tail -1
