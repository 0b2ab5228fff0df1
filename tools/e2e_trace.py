"""Trace where train_single's end-to-end time goes, call by call (C2 shape, 512^3 host volume,
50 iterations), in the order bench.py runs it: one device-resident session first, then the
public train_single with a host Volume, repeated."""
import functools
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
host = L.to_host(vdev)
torch.cuda.synchronize()
events = []


def traced(obj, name):
    f = getattr(obj, name)

    @functools.wraps(f)
    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        events.append((name, 1e3 * (time.perf_counter() - t0)))
        return r
    setattr(obj, name, w)


for n in ("__init__", "run", "status", "pull_params", "log", "close"):
    traced(PT.TrainSession, n)
traced(PV.Volume, "device_data")

if "--after-bench" in sys.argv:  # first the bench's own device-resident run, as in bench.py
    sys.argv = ["bench.py", "--no-cpu-baseline", "--no-inference", "--no-e2e"]
    bench.main()
cfg = PT.TrainConfig(iterations=50, batch_size=1 << 20, delay_start=0, transform_hard_stop_fraction=1.0,
                     plateau_enabled=False, seed=0)
if "--cold" not in sys.argv:
    vol = PV.Volume(dims=dims, data=host)
    m = PM.init_model(PM.ModelConfig(64, 2, (32, 32, 32)), seed=0, vmin=vol.vmin, vmax=vol.vmax)
    PT.train_single(m, vol, cfg)
events.clear()
for rep in range(4):
    vol = PV.Volume(dims=dims, data=host)
    m = PM.init_model(PM.ModelConfig(64, 2, (32, 32, 32)), seed=0, vmin=vol.vmin, vmax=vol.vmax)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    PT.train_single(m, vol, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"rep {rep}: {1e3*dt:.1f} ms -> {50 * (1 << 20) / dt / 1e6:.1f} M pts/s | "
          + ", ".join(f"{n} {t:.1f}" for n, t in events))
    events.clear()

# upload paths: driver pageable copy vs the pinned staging ring
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a = torch.from_numpy(host).to("cuda")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    b = L.to_device(host)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    assert torch.equal(a, b)
    print(f"upload {host.nbytes/2**20:.0f} MiB: pageable {1e3*(t1-t0):.1f} ms, staged {1e3*(t2-t1):.1f} ms")
    del a, b
