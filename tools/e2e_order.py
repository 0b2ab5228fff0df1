"""e2e setup split of train_single (C2 shape, host 512^3 volume) in bench.py's sequence: a device
session first (freed), then train_single calls inside hold_block_cache; per call: setup split,
cudaMalloc / cudaFree counts (torch allocator) and gc collections. """
import gc
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2308_02494_b200 import _lib as L
from paper_2308_02494_b200 import model as PM
from paper_2308_02494_b200 import trainer as PT
from paper_2308_02494_b200 import volume as PV

dims = (512, 512, 512)
vdev = PV.synth_volume_device(dims, [PV.BlobSpec(c, s, a) for c, s, a in bench.BLOBS])
vol0 = PV.Volume.from_device(dims, vdev)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
if os.environ.get("E2E_DEVSESS", "1") == "1":
    m = PM.init_model(PM.ModelConfig(64, 2, (32, 32, 32)), seed=0, vmin=vol0.vmin, vmax=vol0.vmax)
    s = PT.TrainSession(m, vol0, PT.TrainConfig(iterations=30, batch_size=1 << 20, delay_start=0,
                                                transform_hard_stop_fraction=1.0, plateau_enabled=False, seed=0))
    s.run(30)
    torch.cuda.synchronize()
    s.close()
    del s
host = L.to_host(vdev)
cfg = PT.TrainConfig(iterations=K, batch_size=1 << 20, delay_start=0, transform_hard_stop_fraction=1.0,
                     plateau_enabled=False, seed=0)
gcn = [0]
gc.callbacks.append(lambda phase, info: gcn.__setitem__(0, gcn[0] + (phase == "start")))
with PT.hold_block_cache():
    for rep in range(5):
        m = PM.init_model(PM.ModelConfig(64, 2, (32, 32, 32)), seed=0, vmin=vol0.vmin, vmax=vol0.vmax)
        hv = PV.Volume(dims=dims, data=host)
        torch.cuda.synchronize()
        st0 = torch.cuda.memory_stats()
        g0 = gcn[0]
        t0 = time.perf_counter()
        _, log = PT.train_single(m, hv, cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        st1 = torch.cuda.memory_stats()
        d = {k: st1.get(k, 0) - st0.get(k, 0) for k in ("num_device_alloc", "num_device_free", "num_alloc_retries")}
        print(rep, "wall", round(1e3 * dt, 2), "setup", log.setup_ms,
              "loop", round(log.loop_ms, 2), "e2e M/s", round(K * (1 << 20) / dt / 1e6, 1), d, "gc", gcn[0] - g0,
              flush=True)
