#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
APMG_RECON=pp timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_recon_pp -c 1 \
  -o gpurun_out/prof_pp -f python tools/profile_step.py 2 > gpurun_out/ncu_pp.log 2>&1
tail -2 gpurun_out/ncu_pp.log
