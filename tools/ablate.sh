#!/bin/bash
# Timing ablations of the recon kernel (frozen parameters so ablated results cannot change
# later iterations' inputs): builds ab/<name> variants here, runs each on the GPU box.
#   here:     tools/ablate.sh build
#   GPU box:  tools/ablate.sh run
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
VARIANTS="frz:-DAPMG_ABL_FREEZE frz_nored:-DAPMG_ABL_FREEZE_-DAPMG_ABL_NORED frz_nosc:-DAPMG_ABL_FREEZE_-DTC16_ABL_NOSCATTER frz_nogat:-DAPMG_ABL_FREEZE_-DAPMG_ABL_NOGATHER frz_nobump:-DAPMG_ABL_FREEZE_-DTC16_ABL_NOBUMP frz_nomma:-DAPMG_ABL_FREEZE_-DAPMG_ABL_NOMMA frz_nogat_nored:-DAPMG_ABL_FREEZE_-DAPMG_ABL_NOGATHER_-DAPMG_ABL_NORED ${EXTRA_VARIANTS}"
if [ "$1" = build ]; then
  for v in $VARIANTS; do bash tools/ab_build.sh "${v%%:*}" "$(echo "${v#*:}" | tr _ ' ' | sed 's/ABL /ABL_/g;s/APMG /APMG_/g;s/TC16 /TC16_/g')" || exit 1; done
  exit 0
fi
mkdir -p gpurun_out
for r in 1 2; do
  for v in $VARIANTS; do
    n=${v%%:*}
    APMG_LIB="$PWD/ab/$n/libapmg_cuda.so" timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-inference \
      --no-render --no-cpu-baseline 2>>gpurun_out/ablate.err | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$n', round(d['roofline']['ms_per_launch'],4), 'ms recon', round(d['ms_per_step'],4), 'ms step')" \
      | tee -a gpurun_out/ablate.log
  done
done
