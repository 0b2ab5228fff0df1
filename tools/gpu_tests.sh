#!/bin/bash
# GPU pass: the -m gpu suite (durations + the C2 parity prints), smoke, one default bench line.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; free -g >> gpurun_out/host.txt
timeout 300 python tools/peaks.py > gpurun_out/peaks.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_c2_parity.py -m gpu -q -s --durations=0 > gpurun_out/pytest_c2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 --deselect tests/test_gpu_c2_parity.py > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -5 gpurun_out/pytest_c2.log; tail -15 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; head -c 600 gpurun_out/bench.json
