"""Criterion-5 configuration on the GPU (8 grids 8^3 x1, adaptivity volume, batch 2048): final PSNR,
transform stop and the loss trajectory per (seed, adaptive), saved for comparison with the
reference's own run."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_2308_02494_b200 as P
from paper_2308_02494_b200 import model as PM
from paper_2308_02494_b200 import volume as PV

blobs = [PV.BlobSpec(center=(0.45, -0.3, 0.2), sigma=(0.035, 0.035, 0.035)),
         PV.BlobSpec(center=(-0.2, 0.2, -0.1), sigma=(0.6, 0.5, 0.7), amplitude=0.35),
         PV.BlobSpec(center=(0.3, 0.4, 0.5), sigma=(0.45, 0.55, 0.4), amplitude=0.25),
         PV.BlobSpec(center=(-0.5, -0.5, 0.4), sigma=(0.5, 0.4, 0.5), amplitude=0.3)]
vol = PV.synth_volume((64, 64, 64), blobs)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
out = Path("gpurun_out")
out.mkdir(exist_ok=True)
seeds = [int(v) for v in sys.argv[2].split(',')] if len(sys.argv) > 2 else [0]
dets = [bool(int(v)) for v in sys.argv[3].split(',')] if len(sys.argv) > 3 else [False, True]
for seed in seeds:
    for adaptive in (True, False):
        for det in dets:
            m = PM.init_model(PM.ModelConfig(grids=8, channels=1, resolution=(8, 8, 8)), seed=seed, vmin=vol.vmin,
                              vmax=vol.vmax)
            m, log = P.train_single(m, vol, P.TrainConfig(iterations=iters, batch_size=2048, seed=seed,
                                                          train_transforms=adaptive, plateau_enabled=False,
                                                          deterministic=det))
            print(f"seed {seed} adaptive {adaptive} det {det}: psnr {P.psnr(m, vol):.3f} stop "
                  f"{log.transform_stop_iteration} l_rec[-1] {log.l_rec[-1]:.3e}", flush=True)
            np.savez(out / f"gpu_s{seed}_a{int(adaptive)}_d{int(det)}_{iters}.npz", transforms=m.transforms,
                     l_rec=np.array(log.l_rec), l_dens=np.array([np.nan if v is None else v for v in log.l_density]))
