"""Per-phase cycle breakdown of the bf16x3 fused recon kernel (CTA 0, thread 0, tiles 2..14)."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["APMG_TC_STAMPS"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import bench
from paper_2308_02494_b200 import _lib as L
from paper_2308_02494_b200 import model as PM
from paper_2308_02494_b200 import trainer as PT
from paper_2308_02494_b200 import volume as PV

dims = (512, 512, 512)
vdev = PV.synth_volume_device(dims, [PV.BlobSpec(c, s, a) for c, s, a in bench.BLOBS])
vol = PV.Volume.from_device(dims, vdev)
m = PM.init_model(PM.ModelConfig(64, 2, (32, 32, 32)), seed=0, vmin=vol.vmin, vmax=vol.vmax)
cfg = PT.TrainConfig(iterations=10, batch_size=1 << 20, delay_start=0, transform_hard_stop_fraction=1.0,
                     plateau_enabled=False, seed=0)
s = PT.TrainSession(m, vol, cfg)
s.run(4)
torch.cuda.synchronize()
buf = (C.c_longlong * (16 * 12))()
L.check(L.lib().apmg_debug_tc16_phases(buf))
st = np.array(buf[:], dtype=np.int64).reshape(16, 12)[2:15]
names = ["z1 wait", "epilogue 1", "z2 issue + wait", "epi 2 + head + dz2", "dz1 || dW2 (tensor)",
         "dz1 epilogue", "gF || dW1 (tensor)", "gF epilogue", "scatter(t) + encode(t+1)"]
d = np.diff(st[:, :9], axis=1)
nxt = np.roll(st[:, 0], -1)
last = (nxt - st[:, 8])[:-1]
tile = np.diff(st[:, 0])
print(f"cycles per tile (CTA 0): {tile.mean():.0f}")
for i, nm in enumerate(names[:8]):
    print(f"  {nm:28s} {d[:, i].mean():8.0f}  ({100 * d[:, i].mean() / tile.mean():4.1f}%)")
print(f"  {names[8]:28s} {last.mean():8.0f}  ({100 * last.mean() / tile.mean():4.1f}%)")
