#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-render > gpurun_out/bench2.json 2> gpurun_out/bench2.err
python -c "import json; d=json.load(open('gpurun_out/bench2.json')); print(d['value'], d['clocks'], d['e2e']['value'])"
bash tools/upload_sweep.sh > gpurun_out/upload.log 2>&1; cat gpurun_out/upload.log
( time timeout 2400 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
head -c 1500 gpurun_out/bench_ref.json; tail -4 gpurun_out/bench_ref.err
