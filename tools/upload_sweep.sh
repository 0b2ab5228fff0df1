#!/bin/bash
# Host -> device upload of a 512 MiB volume: raw pinned copy (PCIe ceiling) and the staging ring
# at several slot sizes / counts.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
python - <<'PY'
import time, torch
a = torch.empty(512 << 20, dtype=torch.uint8, pin_memory=True)
d = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(2):
    d.copy_(a, non_blocking=True)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    t0 = time.perf_counter(); d.copy_(a, non_blocking=True); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
print(f"pinned H2D 512 MiB: {best*1e3:.1f} ms, {0.5/best:.1f} GiB/s")
PY
for cfg in "16 8" "8 16" "32 8" "4 32" "16 16"; do
  set -- $cfg
  APMG_STAGE_MB=$1 APMG_STAGE_SLOTS=$2 python tools/upload_ab.py
done
