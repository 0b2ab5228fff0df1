"""Host -> device upload throughput of a 512 MiB array through the pinned staging ring."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2308_02494_b200 import _lib as L

a = np.random.default_rng(0).random((512, 512, 512), dtype=np.float32)
L.to_device(a)
best = 1e9
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.to_device(a)
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
print(f"slots {L._STAGE_SLOTS} x {L._STAGE_BYTES >> 20} MiB: {1e3 * best:.1f} ms, {a.nbytes / best / 2**30:.1f} GiB/s")
