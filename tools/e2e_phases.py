"""Where the end-to-end train_single time goes (C2 shape, 512^3 host volume, 50 iterations)."""
import sys
import time
from pathlib import Path

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
host = L.to_host(vdev)
del vdev
torch.cuda.synchronize()


def tic():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(3):
    t0 = tic()
    vol = PV.Volume(dims=dims, data=host)
    t1 = tic()
    dv = vol.device_data()
    t2 = tic()
    m = PM.init_model(PM.ModelConfig(64, 2, (32, 32, 32)), seed=0, vmin=vol.vmin, vmax=vol.vmax)
    t3 = tic()
    cfg = PT.TrainConfig(iterations=50, batch_size=1 << 20, delay_start=0, transform_hard_stop_fraction=1.0,
                         plateau_enabled=False, seed=0)
    s = PT.TrainSession(m, vol, cfg)
    t4 = tic()
    s.run(50)
    t5 = tic()
    s.pull_params()
    lg = s.log()
    s.close()
    t6 = tic()
    print(f"rep {rep}: Volume() {1e3*(t1-t0):.1f} ms, upload {1e3*(t2-t1):.1f} ms, init_model {1e3*(t3-t2):.1f} ms, "
          f"session {1e3*(t4-t3):.1f} ms, run {1e3*(t5-t4):.1f} ms, pull+log+close {1e3*(t6-t5):.1f} ms")


# the bench's e2e call itself
for rep in range(3):
    vol = PV.Volume(dims=dims, data=host)
    m = PM.init_model(PM.ModelConfig(64, 2, (32, 32, 32)), seed=0, vmin=vol.vmin, vmax=vol.vmax)
    cfg = PT.TrainConfig(iterations=50, batch_size=1 << 20, delay_start=0, transform_hard_stop_fraction=1.0,
                         plateau_enabled=False, seed=0)
    t0 = tic()
    _, lg = PT.train_single(m, vol, cfg)
    t1 = tic()
    print(f"train_single e2e rep {rep}: {1e3*(t1-t0):.1f} ms -> {50 * (1 << 20) / (t1 - t0) / 1e6:.1f} M pts/s")
