"""Time the renderer field-query path: one C2-shaped model (64 grids 32^3 x2), a 512^2 frame,
128 samples per ray (33.5 M field queries)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2308_02494_b200 import model as PM
from paper_2308_02494_b200 import render as PR

m = PM.init_model(PM.ModelConfig(64, 2, (32, 32, 32)), seed=0, vmin=0.0, vmax=1.0)
rng = np.random.default_rng(0)
m.grids[:] = rng.normal(scale=0.3, size=m.grids.shape).astype(np.float32)
size = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cam = PR.Camera(eye=(1.6, 1.1, 2.4), look_at=(0, 0, 0), width=size, height=size)
tf = PR.TransferFunction(opacity_points=[(0.0, 0.0), (0.5, 0.05), (1.0, 0.6)])
for early in (0.99, None):
    cfg = PR.RenderConfig(samples_per_ray=128, early_exit_alpha=early)
    PR.render_frame(PR.ModelField(m), cam, tf, cfg)  # warm-up
    torch.cuda.synchronize()
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        img = PR.render_frame(PR.ModelField(m), cam, tf, cfg)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    q = size * size * 128
    print(f"{size}^2 x 128 early={early}: {1e3 * dt:.1f} ms/frame, {q / dt / 1e9:.2f} G field queries/s "
          f"(upper bound: all rays hit), mean alpha {img[..., 3].mean():.3f}")

# per-kernel split of one frame (CUDA events around every launch) and the host-side phases
import bench  # noqa: E402
from paper_2308_02494_b200 import _lib as L  # noqa: E402
for early in (0.99, None):
    cfg = PR.RenderConfig(samples_per_ray=128, early_exit_alpha=early)
    L.lib().apmg_kernel_timing_enable(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    origin, dirs = PR.generate_rays(cam)
    t1 = time.perf_counter()
    rgba, evals = PR._render_rays(PR.ModelField(m), origin, dirs, tf, cfg)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    tab = bench.kernel_table()
    L.lib().apmg_kernel_timing_enable(0)
    print(f"early={early}: generate_rays {1e3 * (t1 - t0):.1f} ms, _render_rays {1e3 * (t2 - t1):.1f} ms, "
          f"evals {evals / (size * size * 128):.2f} of all samples")
    for k, v in sorted(tab.items(), key=lambda kv: -kv[1]["total_ms"]):
        print(f"   {k:24s} {v['total_ms']:8.2f} ms  x{v['launches']}")
