"""Per-phase cycle breakdown of the tensor-core lattice sweep (CTA 0, thread 0, tiles 2..14)."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["APMG_INFER_STAMPS"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import bench
from paper_2308_02494_b200 import _lib as L

bench.bench_inference(dims=(256, 256, 256))
torch.cuda.synchronize()
buf = (C.c_longlong * (16 * 8))()
L.check(L.lib().apmg_debug_infer_phases(buf))
st = np.array(buf[:], dtype=np.int64).reshape(16, 8)[2:15]
cols = [0, 2, 3, 4]
names = ["encode + sync", "z1 issue, coords(t+1), head(t-1)", "epi1 + z2 issue", "loop back"]
nxt = np.roll(st[:, 0], -1)
d = np.stack([st[:, 2] - st[:, 0], st[:, 3] - st[:, 2], st[:, 4] - st[:, 3], nxt - st[:, 4]], axis=1)[:-1]
tile = np.diff(st[:, 0])
print(f"cycles per tile (CTA 0): {tile.mean():.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:34s} {d[:, i].mean():8.0f}  ({100 * d[:, i].mean() / tile.mean():4.1f}%)")
