cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2 || exit 1
ROUNDS=3 bash tools/ab_bench.sh mbarwait > /dev/null 2>&1
cat gpurun_out/ab.log
for lib in "" "$PWD/ab/mbarwait/libapmg_cuda.so"; do
  APMG_DETERMINISTIC=1 APMG_LIB="$lib" timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-inference --no-render --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('DET lib=${lib##*/ab/}', round(d['value']/1e6,1), 'M pts/s', round(d['roofline']['ms_per_launch'],4), 'ms recon')"
done
timeout 900 python -m pytest tests/test_gpu_c2_parity.py -m gpu -q -s 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_c2_parity.py > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
