#!/bin/bash
# A/B of library builds on the GPU box: alternates the default build and each ab/<name> variant,
# ROUNDS times, printing the device-timed train points/s of the C2 step for each run.
#   tools/ab_bench.sh name1 [name2 ...]        (ROUNDS=3 STEPS=20 by default)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
ROUNDS=${ROUNDS:-3}; STEPS=${STEPS:-20}
for r in $(seq "$ROUNDS"); do
  for v in default "$@"; do
    if [ "$v" = default ]; then lib=""; else lib="$PWD/ab/$v/libapmg_cuda.so"; fi
    APMG_LIB=$lib timeout 300 python bench.py --steps "$STEPS" --warmup 5 --no-e2e --no-inference --no-render \
      --no-cpu-baseline 2>>gpurun_out/ab.err | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,1), 'M pts/s', {k: round(v,4) for k,v in list(d['kernel_share'].items())[:2]}, round(d['roofline']['ms_per_launch'],4), 'ms recon')" \
      | tee -a gpurun_out/ab.log
  done
done
