#!/bin/bash
# Inference / render A/B: the default against ab/<name> builds or VAR=value switches (args), two
# rounds, then the sweep / render / forward tests.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for r in 1 2; do for v in default "$@"; do
lib=""; envs=()
if [[ "$v" == *=* ]]; then envs=("$v"); elif [ "$v" != default ]; then lib="$PWD/ab/$v/libapmg_cuda.so"; fi
env APMG_LIB="$lib" "${envs[@]}" timeout 240 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['inference']['value']/1e9,3), 'Gvox/s', round(d['inference']['ms_per_sweep'],2), 'render', round(d['render'].get('ms_per_frame'),2))"
done; done
timeout 900 python -m pytest tests -m gpu -q -x -k "lattice or sweep or render or forward or infer or decomposed or psnr" 2>&1 | tail -1
