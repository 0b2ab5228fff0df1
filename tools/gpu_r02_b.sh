#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
APMG_RECON=pp timeout 600 python -m pytest tests/test_gpu_c2_parity.py tests/test_gpu_parity.py -m gpu -q -x -s \
  -k "c2 or recon_tensor_core or full_size or fused_density or gridx or deterministic or c1_psnr_parity_60 or train_small or cell_volume" \
  > gpurun_out/pytest_pp.log 2>&1
tail -4 gpurun_out/pytest_pp.log; grep -E "^C2 " gpurun_out/pytest_pp.log
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_mr.log 2>&1; tail -2 gpurun_out/pytest_mr.log
ROUNDS=3 timeout 900 bash tools/ab_bench.sh APMG_RECON=pp
