#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for r in 1 2; do
  for v in default fxcap1 fxcap7; do
    lib=""; [ "$v" != default ] && lib="$PWD/ab/$v/libapmg_cuda.so"
    APMG_DETERMINISTIC=1 APMG_LIB="$lib" timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-inference \
      --no-render --no-cpu-baseline 2>>gpurun_out/ab.err | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('det $v', round(d['value']/1e6,1), 'M pts/s', round(d['roofline']['ms_per_launch'],4), 'ms recon')"
  done
done
for cfg in "32 8" "32 16" "64 8" "32 12" "64 16"; do
  set -- $cfg
  APMG_STAGE_MB=$1 APMG_STAGE_SLOTS=$2 python tools/upload_ab.py
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "deterministic" > gpurun_out/pytest_det.log 2>&1; tail -2 gpurun_out/pytest_det.log
