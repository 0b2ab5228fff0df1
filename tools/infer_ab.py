"""C3 lattice sweep throughput (bench_inference) and the renderer frame time, for quick A/Bs."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

r = bench.bench_inference()
print("C3", round(r["value"] / 1e9, 3), "G vox/s", round(r["ms_per_sweep"], 1), "ms")
f = bench.bench_render()
print("render", round(f["ms_per_frame"], 2), "ms/frame")
