#!/bin/bash
# One default bench line (and the e2e split) on the GPU box: gpurun_out/bench.json
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print(round(d['value']/1e6,1), 'M pts/s', 'e2e', round(d['e2e']['value']/1e6,1), d['e2e'].get('setup_ms'), d['e2e'].get('setup_split_ms'), d['e2e'].get('loop_ms'), d['e2e'].get('wall_ms'))
print('cpu', d.get('cpu_baseline')); print('clocks', d.get('clocks'))"
