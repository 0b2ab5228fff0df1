cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
ROUNDS=3 bash tools/ab_bench.sh d4 APMG_DENS_X4=0 > /dev/null 2>&1
cat gpurun_out/ab.log
timeout 900 python -m pytest tests/test_gpu_c2_parity.py -m gpu -q -s 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -x -k "density or train" --deselect tests/test_gpu_c2_parity.py 2>&1 | tail -2
