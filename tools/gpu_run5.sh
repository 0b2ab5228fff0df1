cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
ROUNDS=3 bash tools/ab_bench.sh oldsc pk_noround old_round > /dev/null 2>&1
cat gpurun_out/ab.log
APMG_LIB=$PWD/ab/oldsc/libapmg_cuda.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_recon_tc16 -s 2 -c 1 \
  -o gpurun_out/prof_src -f python tools/profile_step.py 3 > gpurun_out/ncu_src.log 2>&1
tail -2 gpurun_out/ncu_src.log
