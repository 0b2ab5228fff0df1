"""Short C2 training run for profiling: W warm-up + K timed iterations at batch 2^20."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2308_02494_b200 import model as PM
from paper_2308_02494_b200 import trainer as PT
from paper_2308_02494_b200 import volume as PV

BLOBS = [((0.45, -0.3, 0.2), (0.035, 0.035, 0.035), 1.0), ((-0.2, 0.2, -0.1), (0.6, 0.5, 0.7), 0.35),
         ((0.3, 0.4, 0.5), (0.45, 0.55, 0.4), 0.25), ((-0.5, -0.5, 0.4), (0.5, 0.4, 0.5), 0.3)]
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dims = (512, 512, 512)
vdev = PV.synth_volume_device(dims, [PV.BlobSpec(c, s, a) for c, s, a in BLOBS])
vol = PV.Volume.from_device(dims, vdev)
m = PM.init_model(PM.ModelConfig(64, 2, (32, 32, 32)), seed=0, vmin=vol.vmin, vmax=vol.vmax)
cfg = PT.TrainConfig(iterations=iters, batch_size=1 << 20, delay_start=0, transform_hard_stop_fraction=1.0,
                     plateau_enabled=False, seed=0)
s = PT.TrainSession(m, vol, cfg)
s.run(iters)
torch.cuda.synchronize()
print("ran", s.status())
