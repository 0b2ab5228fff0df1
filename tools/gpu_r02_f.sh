#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c2_parity.py tests/test_gpu_parity.py -m gpu -q -x -s -k "c2 or density or recon or train or fused" > gpurun_out/pytest_f.log 2>&1; tail -2 gpurun_out/pytest_f.log; grep "^C2" gpurun_out/pytest_f.log
ROUNDS=2 timeout 900 bash tools/ab_bench.sh
python - <<'PY'
import json, subprocess, sys
out = subprocess.run([sys.executable, "bench.py", "--steps", "20", "--warmup", "5", "--no-e2e", "--no-inference", "--no-render", "--no-cpu-baseline"], capture_output=True, text=True).stdout
d = json.loads(out)
print({k: v for k, v in d["roofline"]["other_kernels"].items()}, d["kernel_share"])
PY
