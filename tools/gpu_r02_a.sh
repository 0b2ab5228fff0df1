#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
df -h /tmp > gpurun_out/df.txt
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -m gpu -q -x --durations=10 \
  --deselect tests/test_gpu_parity.py::test_train_c1_300_baseline_parity > gpurun_out/pytest_a.log 2>&1
tail -3 gpurun_out/pytest_a.log
ROUNDS=3 timeout 900 bash tools/ab_bench.sh spin
APMG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-inference \
  > gpurun_out/bench_c4_gloo.json 2> gpurun_out/bench_c4_gloo.err
tail -c 1500 gpurun_out/bench_c4_gloo.json; grep -i "error\|Traceback" gpurun_out/bench_c4_gloo.err | head -5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_recon_tc16 -c 1 \
  -o gpurun_out/prof_tc16_r02a -f python tools/profile_step.py 2 > gpurun_out/ncu_a.log 2>&1
tail -2 gpurun_out/ncu_a.log
