#!/bin/bash
# One GPU pass: parity suite, smoke, default bench, short reference arm, ncu launch list and a
# `--set full` capture of the step's kernels.  Outputs land in gpurun_out/ (merged back by gpurun).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
APMG_REF_BUDGET_S=30 timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-inference --no-render > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_recon_tc16|k_dens_grad32c|k_dens_rho32|k_sample_sorted|k_bucket_scatter|k_batch_keys|k_adam_train|k_infer_tc" \
  -c 8 -o gpurun_out/prof_$TAG -f python tools/profile_step.py 2 > gpurun_out/ncu_f.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.json gpurun_out/bench_ref.json
tail -2 gpurun_out/ncu_f.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_infer_tc -c 1 \
  -o gpurun_out/prof_infer_$TAG -f python tools/profile_infer.py 512 512 512 > gpurun_out/ncu_infer.log 2>&1
tail -1 gpurun_out/ncu_infer.log
