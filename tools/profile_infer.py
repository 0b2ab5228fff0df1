"""One C3-shaped lattice sweep (1024^3, PSNR mode) for profiling."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench

r = bench.bench_inference(dims=tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (1024, 1024, 1024))
torch.cuda.synchronize()
print(r)
