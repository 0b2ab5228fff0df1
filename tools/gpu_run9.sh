cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
ROUNDS=3 bash tools/ab_bench.sh APMG_ADAM_SIDE=0 > /dev/null 2>&1
cat gpurun_out/ab.log
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_c2_parity.py > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
