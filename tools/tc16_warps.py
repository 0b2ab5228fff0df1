"""Per-warp phase timeline of the bf16x3 fused recon kernel (CTA 0, all 16 warps, tiles 2..14):
for every stamp point, the mean over tiles of (warp's stamp - tile start), so the spread across
warps shows who the barriers wait for."""
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
buf = (C.c_longlong * (16 * 16 * 16))()
L.check(L.lib().apmg_debug_tc16_warp_phases(buf))
st = np.array(buf[:], dtype=np.int64).reshape(16, 16, 16)[2:15].astype(np.float64)  # [tile][warp][point]
t0 = st[:, :, 0].min(axis=1)[:, None]  # tile start: earliest warp at the loop top
rel = st - t0[:, :, None]
names = {0: "loop top", 1: "z1 done", 2: "epi1 barrier", 13: "scatter u3 done", 3: "z2 done",
         4: "epi2 barrier", 14: "scatter u4 done", 5: "dz1||dW2 done", 6: "dz1 epi barrier",
         15: "scatter u5-7 done", 7: "gF||dW1 done+sync", 8: "gF epi sync", 9: "enc group0 done",
         10: "z1a barrier", 11: "enc group1 done", 12: "encode sync"}
order = [0, 1, 2, 13, 3, 4, 14, 5, 6, 15, 7, 8, 9, 10, 11, 12]
tile = np.diff(st[:, 0, 0]).mean()
print(f"cycles per tile (CTA 0): {tile:.0f}")
print(f"{'point':22s} " + " ".join(f"w{w:<5d}" for w in range(16)))
for k in order:
    v = rel[:, :, k].mean(axis=0)
    print(f"{k:2d} {names[k]:19s} " + " ".join(f"{x:6.0f}" for x in v))
