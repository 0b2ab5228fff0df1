cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
ROUNDS=3 bash tools/ab_bench.sh i4b2 i2b2 > /dev/null 2>&1
cat gpurun_out/ab.log
