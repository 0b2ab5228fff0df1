#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fused_batch or c2 or cell_volume or train_c1_psnr_parity_60" > gpurun_out/pytest_e.log 2>&1; tail -2 gpurun_out/pytest_e.log
ROUNDS=3 timeout 900 bash tools/ab_bench.sh cap2 cap3 APMG_FUSED_BATCH=0
