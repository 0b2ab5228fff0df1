cd $GRAFT_REPO_ROOT
ROUNDS=3 bash tools/ab_bench.sh oldsc > /dev/null 2>&1
cat gpurun_out/ab.log
for r in 1 2; do
 for lib in "" "$PWD/ab/oldsc/libapmg_cuda.so"; do
  APMG_DETERMINISTIC=1 APMG_LIB="$lib" timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-inference --no-render --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('DET lib=${lib##*/ab/}', round(d['value']/1e6,1), 'M pts/s', round(d['roofline']['ms_per_launch'],4), 'ms recon')"
 done
done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
