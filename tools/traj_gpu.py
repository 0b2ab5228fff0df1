"""Transform trajectory of the criterion-5 model with the density step from iteration 2 (80
iterations, batch 2048) on the GPU, against a reference run stored in tools/_tmp/ref_traj.npz."""
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
ref = np.load("tools/_tmp/ref_traj.npz")
for det in (True,):
    m = PM.init_model(PM.ModelConfig(grids=8, channels=1, resolution=(8, 8, 8)), seed=0, vmin=vol.vmin, vmax=vol.vmax)
    tfs = []
    m, log = P.train_single(m, vol, P.TrainConfig(iterations=80, batch_size=2048, seed=0, delay_start=2,
                                                  plateau_enabled=False, deterministic=det),
                            on_iteration=lambda it, mm: tfs.append(mm.transforms.copy()))
    tfs = np.array(tfs)
    for it in (0, 1, 2, 3, 4, 5, 8, 12, 16, 20, 30, 40, 60, 79):
        d = np.abs(tfs[it] - ref["tfs"][it]).max()
        moved = np.abs(ref["tfs"][it] - ref["tfs"][0]).max()
        print(f"it {it:3d}: l_rec gpu {log.l_rec[it]:.6e} ref {ref['l_rec'][it]:.6e} | l_dens gpu "
              f"{log.l_density[it] if log.l_density[it] is not None else float('nan'):.6e} ref {ref['l_dens'][it]:.6e} "
              f"| max|dT| {d:.2e} (ref moved {moved:.2e})")
