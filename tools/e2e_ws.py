"""Where TrainSession setup time goes inside bench.py's e2e calls: workspace allocation (torch
caching allocator: new segments = cudaMalloc) and the library's size queries, per call."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2308_02494_b200 import _lib as L

orig_ws = L.workspace


def ws(n):
    torch.cuda.synchronize()
    s0 = torch.cuda.memory_stats().get("segment.all.allocated", 0)
    t0 = time.perf_counter()
    r = orig_ws(n)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    s1 = torch.cuda.memory_stats().get("segment.all.allocated", 0)
    print(f"  workspace {n / 2**30:.3f} GiB: {1e3 * (t1 - t0):.2f} ms, new segments {s1 - s0}", file=sys.stderr, flush=True)
    return r


L.workspace = ws
lib = L.lib()
orig_vb = lib.apmg_train_volume_bytes


class Wrap:
    def __getattr__(self, k):
        f = getattr(lib, k)
        if k not in ("apmg_train_volume_bytes", "apmg_train_workspace_bytes", "apmg_train_create"):
            return f

        def g(*a):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = f(*a)
            print(f"  {k}: {1e3 * (time.perf_counter() - t0):.2f} ms", file=sys.stderr, flush=True)
            return r
        return g


L.lib = lambda: Wrap()
sys.argv = ["bench.py", "--steps", "20", "--warmup", "5", "--no-inference", "--no-render", "--no-cpu-baseline"]
bench.main()
