"""Brick ingest: a ghost extent of a raw float32 volume file to the GPU -- load_subvolume (memmap
copy, then upload) vs load_subvolume_device (memmap pieces -> pinned ring -> device)."""
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2308_02494_b200 import volume as PV

n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
with tempfile.TemporaryDirectory(dir="/tmp") as td:
    raw = Path(td) / "v.raw"
    rng = np.random.default_rng(0)
    with open(raw, "wb") as f:
        for z in range(n):
            f.write(rng.random((n, n), dtype=np.float32).tobytes())
    hdr = PV.VolumeHeader(dims=(n, n, n))
    h = n // 2 + 1
    ext = PV.Extent(lo=(n - h, 0, n // 4), hi=(n - 1, h - 1, n // 4 + h - 1))
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a = PV.load_subvolume(raw, hdr, ext)
        a.device_data()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        b = PV.load_subvolume_device(raw, hdr, ext)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        mb = h ** 3 * 4 / 2 ** 20
        print(f"{h}^3 extent ({mb:.0f} MiB) of a {n}^3 file: load_subvolume + upload {1e3 * (t1 - t0):.0f} ms, "
              f"streamed {1e3 * (t2 - t1):.0f} ms ({mb / 1024 / (t2 - t1):.1f} GiB/s)")
    assert torch.equal(a.device_data(), b.device_data())
