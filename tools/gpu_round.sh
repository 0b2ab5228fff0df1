#!/bin/bash
# One GPU pass: parity suite, smoke, default bench, reference arm, ncu launch list and a
# `--set full` capture of the step's kernels + the lattice sweep.  Outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 2400 python -m pytest tests -m gpu -q -x -s --durations=20 > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ -z "$NO_REF" ]; then
  timeout 2400 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-inference --no-render > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_recon_tc16|k_dens_grad32c|k_sample_sorted|k_bucket_scatter|k_batch_keys|k_adam_train" \
  -c 6 -o gpurun_out/prof_$TAG -f python tools/profile_step.py 2 > gpurun_out/ncu_f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_infer_tc -c 1 \
  -o gpurun_out/prof_infer_$TAG -f python tools/profile_infer.py 512 512 512 > gpurun_out/ncu_infer.log 2>&1
grep -E "passed|failed|C1-300|C2 " gpurun_out/pytest_gpu.log | tail -8; tail -1 gpurun_out/smoke.log
head -c 400 gpurun_out/bench.json; echo; head -c 600 gpurun_out/bench_ref.json; echo
tail -1 gpurun_out/ncu_f.log; tail -1 gpurun_out/ncu_infer.log
