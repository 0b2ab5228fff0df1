"""Diagnostic: GPU train_single vs the CPU oracle on the C1 parity config, per-iteration
parameter divergence (per-tensor relative norm) at selected iterations."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from oracle import apmg_oracle as O
import paper_2308_02494_b200 as P
from paper_2308_02494_b200 import model as PM
from paper_2308_02494_b200 import volume as PV

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 2 ** 14
snap_at = {0, 1, 2, 4, 9, 49, 50, 51, 55, 60, 100, 150, 199}
blobs = [((0.45, -0.3, 0.2), (0.035,) * 3, 1.0), ((-0.2, 0.2, -0.1), (0.6, 0.5, 0.7), 0.35),
         ((0.3, 0.4, 0.5), (0.45, 0.55, 0.4), 0.25), ((-0.5, -0.5, 0.4), (0.5, 0.4, 0.5), 0.3)]
vol_np = O.synth_volume((128, 128, 128), blobs)
vol = PV.Volume(dims=(128, 128, 128), data=vol_np)
keys = ("transforms", "grids", "w1", "w2", "w3")
gpu_snaps, cpu_snaps = {}, {}
m = PM.init_model(PM.ModelConfig(64, 2, (32, 32, 32)), seed=0, vmin=vol.vmin, vmax=vol.vmax)
cfg = P.TrainConfig(iterations=iters, batch_size=batch, delay_start=min(50, iters - 1), seed=0, plateau_enabled=False)
_, glog = P.train_single(m, vol, cfg, on_iteration=lambda it, mm: gpu_snaps.update(
    {it: {k: getattr(mm, k).copy() for k in keys}}) if it in snap_at else None)
prm = O.init_params(64, 2, (32, 32, 32), seed=0, vmin=vol.vmin, vmax=vol.vmax)
ocfg = O.LoopConfig(iterations=iters, batch_size=batch, delay_start=min(50, iters - 1), seed=0, plateau_enabled=False)
olog = O.train_single(prm, vol_np, ocfg, on_iteration=lambda it, p: cpu_snaps.update(
    {it: {k: getattr(p, k).copy() for k in keys}}) if it in snap_at else None)
for it in sorted(gpu_snaps):
    if it not in cpu_snaps:
        continue
    rel = {k: float(np.linalg.norm(gpu_snaps[it][k].astype(np.float64) - cpu_snaps[it][k]) /
                   max(np.linalg.norm(cpu_snaps[it][k].astype(np.float64)), 1e-30)) for k in keys}
    print(f"it {it:4d} l_rec gpu {glog.l_rec[it]:.6e} cpu {olog.l_rec[it]:.6e} "
          f"ld gpu {glog.l_density[it]} cpu {olog.l_density[it]} | " +
          " ".join(f"{k}={v:.2e}" for k, v in rel.items()), flush=True)
print("stop", glog.transform_stop_iteration, olog.transform_stop_iteration)
print("psnr gpu", P.psnr(m, vol), "cpu", O.psnr(lambda q: O.forward(prm, q), vol_np))
