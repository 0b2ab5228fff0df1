#!/bin/bash
# A/B an environment switch on the default bench: tools/bench_ab.sh VAR "v1 v2 ..." [bench args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
var=$1; vals=$2; shift 2
for v in $vals; do
  env "$var=$v" python bench.py --no-cpu-baseline --no-inference --no-render "$@" 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read())
e = d.get('e2e') or {}
print('$var=$v', round(d['value'] / 1e6, 1), 'M/s', round(d['ms_per_step'], 4), 'ms', 'e2e', round((e.get('value') or 0) / 1e6, 1),
      {k: v for k, v in list(d.get('kernel_share', {}).items())[:4]}, 'sum', round(sum(d.get('kernel_share', {}).values()), 4))
if '$AB_ALL' == '1': print('   ', d.get('kernel_share'))"
done
