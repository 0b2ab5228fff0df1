import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2308_02494_b200 import _lib as L
def run(cfg, K, N, flags=0, split=1):
    M = 128 if cfg >= 2 else 64
    rng = np.random.default_rng(cfg)
    if cfg in (0, 3):
        A = rng.normal(size=(M, K)).astype(np.float32); B = rng.normal(size=(N, K)).astype(np.float32); ref = A.astype(np.float64) @ B.T
    elif cfg == 1:
        A = rng.normal(size=(M, K)).astype(np.float32); B = rng.normal(size=(K, N)).astype(np.float32); ref = A.astype(np.float64) @ B
    else:
        A = rng.normal(size=(K, 128)).astype(np.float32); B = rng.normal(size=(K, N)).astype(np.float32); ref = A.astype(np.float64).T @ B
    a_d, b_d = L.to_device(A), L.to_device(B)
    d = L.zeros((M, N), np.float32)
    L.check(L.lib().apmg_debug_umma_gemm(cfg | flags, K, N, split, L.ptr(a_d), L.ptr(b_d), L.ptr(d), L.stream_handle()))
    D = L.to_host(d)
    print(f"cfg {cfg} K {K} N {N} flags {flags} split {split}: err {np.abs(D - ref).max() / np.abs(ref).max():.2e} Dabsmax {np.abs(D).max():.3g} D[0,0:3] {D[0,0:3]} D[1,0:2] {D[1,0:2]} ref[0,0:3] {ref[0,0:3]}")
run(1, 8, 16, 131072, 0); run(1, 64, 128, 131072, 1); run(2, 64, 64, 131072, 1); run(2, 64, 80, 131072, 1)
run(1, 8, 16, 0, 0)
run(0, 8, 16, 0, 0)
run(2, 8, 16, 0, 0)
