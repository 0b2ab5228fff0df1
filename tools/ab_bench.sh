#!/bin/bash
# A/B on the GPU box: alternates the default build/configuration with each variant, ROUNDS times,
# printing the device-timed train points/s of the C2 step.  A variant is either the name of an
# ab/<name>/libapmg_cuda.so build (tools/ab_build.sh) or VAR=value (an environment switch).
#   tools/ab_bench.sh spin APMG_RECON=pp        (ROUNDS=3 STEPS=20 by default)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
ROUNDS=${ROUNDS:-3}; STEPS=${STEPS:-20}
for r in $(seq "$ROUNDS"); do
  for v in default "$@"; do
    lib=""; envs=()
    if [[ "$v" == *=* ]]; then envs=("$v"); elif [ "$v" != default ]; then lib="$PWD/ab/$v/libapmg_cuda.so"; fi
    env APMG_LIB="$lib" "${envs[@]}" timeout 300 python bench.py --steps "$STEPS" --warmup 5 --no-e2e --no-inference \
      --no-render --no-cpu-baseline 2>>gpurun_out/ab.err | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,1), 'M pts/s', {k: round(v,4) for k,v in list(d['kernel_share'].items())[:2]}, round(d['roofline']['ms_per_launch'],4), 'ms recon', 'l_rec', d['final_l_rec'])" \
      | tee -a gpurun_out/ab.log
  done
done
