"""Stage cost breakdown of the fused recon kernel: re-time the C2 step with stages disabled
(APMG_TC_SKIP bitmask: 1 scatter, 2 backward MMAs, 4 encoder gathers).  Results of the
disabled runs are wrong by construction; only the kernel times are meaningful."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r'''
import sys, json, torch
sys.path.insert(0, sys.argv[1])
import bench
from paper_2308_02494_b200 import _lib as L, model as PM, trainer as PT, volume as PV
dims = (512, 512, 512)
vdev = PV.synth_volume_device(dims, [PV.BlobSpec(c, s, a) for c, s, a in bench.BLOBS])
vol = PV.Volume.from_device(dims, vdev)
m = PM.init_model(PM.ModelConfig(64, 2, (32, 32, 32)), seed=0, vmin=vol.vmin, vmax=vol.vmax)
cfg = PT.TrainConfig(iterations=30, batch_size=1 << 20, delay_start=0, transform_hard_stop_fraction=1.0,
                     plateau_enabled=False, seed=0)
s = PT.TrainSession(m, vol, cfg)
s.run(5); torch.cuda.synchronize()
L.lib().apmg_kernel_timing_enable(1)
s.run(20); torch.cuda.synchronize()
t = bench.kernel_table()
print(json.dumps({k: v["total_ms"] / v["launches"] for k, v in t.items()}))
'''
if __name__ == "__main__":
    res = {}
    for skip in [int(v) for v in (sys.argv[1:] or ["0", "1", "2", "4", "3", "5", "7"])]:
        env = dict(os.environ, APMG_TC_SKIP=str(skip))
        env.update({k: v for k, v in (kv.split("=") for kv in os.environ.get("EXTRA", "").split() if kv)})
        out = subprocess.run([sys.executable, "-c", CHILD, str(ROOT)], env=env, capture_output=True, text=True)
        try:
            t = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            print(out.stdout[-2000:], out.stderr[-2000:])
            continue
        res[skip] = t
        rk = [k for k in t if k.startswith("recon")]
        print(skip, {k: round(t[k], 3) for k in rk}, "step", round(sum(t.values()), 3), flush=True)
    print(json.dumps(res))
