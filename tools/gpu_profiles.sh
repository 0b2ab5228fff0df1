#!/bin/bash
# ncu evidence for one tag: the launch list of a bench-shaped run (shares), a --set full capture of
# the C2 step kernels and of the lattice sweep.  Summarise here with:
#   python tools/make_profiles.py TAG gpurun_out/launches_TAG.csv gpurun_out/prof_TAG.ncu-rep
#   python tools/make_profiles.py TAG_infer "" gpurun_out/prof_infer_TAG.ncu-rep
#   python tools/traffic_json.py TAG TAG TAG_infer ; python tools/sass_counts.py TAG
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r02b}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-inference --no-render > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_recon_tc16|k_dens_grad32c|k_sample_sorted|k_bucket_scatter|k_batch_keys|k_adam_train|k_dens_target" \
  -c 7 -o gpurun_out/prof_$TAG -f python tools/profile_step.py 2 > gpurun_out/ncu_f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_infer_tc -c 1 \
  -o gpurun_out/prof_infer_$TAG -f python tools/profile_infer.py 512 512 512 > gpurun_out/ncu_infer.log 2>&1
tail -1 gpurun_out/ncu_l.log; tail -1 gpurun_out/ncu_f.log; tail -1 gpurun_out/ncu_infer.log; ls -la gpurun_out/*$TAG*
