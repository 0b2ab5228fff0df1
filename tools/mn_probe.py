"""Probe MN-major kind::tf32 operand descriptors through the umma self-test kernel."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from paper_2308_02494_b200 import _lib as L


def run(cfg, flags, K, N, split3, seed=0):
    rng = np.random.default_rng(seed + 17 * cfg + K + N)
    M = 128 if cfg >= 2 else 64
    if cfg in (0, 3, 4):
        A = rng.normal(size=(M, K)).astype(np.float32); B = rng.normal(size=(N, K)).astype(np.float32)
        ref = A.astype(np.float64) @ B.astype(np.float64).T
    elif cfg == 1:
        A = rng.normal(size=(M, K)).astype(np.float32); B = rng.normal(size=(K, N)).astype(np.float32)
        ref = A.astype(np.float64) @ B.astype(np.float64)
    else:
        A = rng.normal(size=(K, 128)).astype(np.float32); B = rng.normal(size=(K, N)).astype(np.float32)
        ref = A.astype(np.float64).T @ B.astype(np.float64)
    d = L.zeros((M, N), np.float32)
    a_d, b_d = L.to_device(A), L.to_device(B)
    L.check(L.lib().apmg_debug_umma_gemm(cfg | flags, K, N, split3, L.ptr(a_d), L.ptr(b_d), L.ptr(d),
                                         L.stream_handle()), "umma")
    got = L.to_host(d).astype(np.float64)
    return float(np.max(np.abs(got - ref)) / np.max(np.abs(ref))), float(np.abs(got).max())


for cfg, flags_list in ((4, (0,)), (1, (0,))):
    for flags in flags_list:
        for K, N in ((64, 64), (8, 16), (64, 128), (32, 64)):
            try:
                print(cfg, flags, K, N, run(cfg, flags, K, N, 1), run(cfg, flags, K, N, 0), flush=True)
            except Exception as e:
                print(cfg, flags, K, N, "ERR", e, flush=True)
