#!/bin/bash
# A/B: xy-quad grid copy (256-bit gathers) vs x-pair, plus the quad path's parity tests
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 bash tools/bench_ab.sh APMG_GRIDQ "0 1 0 1" --steps 30 --warmup 5 --no-e2e > gpurun_out/quad_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_c2_parity.py -m gpu -q -s > gpurun_out/pytest_c2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_c2_parity.py > gpurun_out/pytest_gpu.log 2>&1
cat gpurun_out/quad_ab.log; tail -3 gpurun_out/pytest_c2.log; tail -8 gpurun_out/pytest_gpu.log
