"""tcgen05 bring-up: the CM-layout operand staging, smem/instruction descriptors,
kind::tf32 MMA and TMEM readback used by the fused MLP, one GEMM per config,
against float64 numpy (3xTF32 split and single TF32)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2308_02494_b200 import _lib as L  # noqa: E402


def run(cfg, K, N, split3, seed=0):
    rng = np.random.default_rng(seed + 17 * cfg + K + N)
    M = 128 if cfg >= 2 else 64
    if cfg in (0, 3, 4):
        A = rng.normal(size=(M, K)).astype(np.float32)
        B = rng.normal(size=(N, K)).astype(np.float32)
        ref = A.astype(np.float64) @ B.astype(np.float64).T
    elif cfg == 1:
        A = rng.normal(size=(M, K)).astype(np.float32)
        B = rng.normal(size=(K, N)).astype(np.float32)
        ref = A.astype(np.float64) @ B.astype(np.float64)
    else:
        A = rng.normal(size=(K, 128)).astype(np.float32)
        B = rng.normal(size=(K, N)).astype(np.float32)
        ref = A.astype(np.float64).T @ B.astype(np.float64)
    d = L.zeros((M, N), np.float32)
    a_d, b_d = L.to_device(A), L.to_device(B)  # both alive at launch (no allocator reuse)
    L.check(L.debug_lib().apmg_debug_umma_gemm(cfg, K, N, split3, L.ptr(a_d), L.ptr(b_d), L.ptr(d),
                                         L.stream_handle()), "umma")
    got = L.to_host(d).astype(np.float64)
    return float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))


# K-major A and B from smem (the forward products of the fused recon kernel): M=64 and M=128
# accumulators; cfg 4: A from tensor memory (the kernel's dz1^T and gF^T products, whose
# transposed weights stay resident in TMEM).  MN-major kind::tf32 smem operands need the
# 128B/32B-atom swizzle (configs 1-2 of the self-test use SWIZZLE_NONE and read zeros), so the
# kernel does not issue them.
@pytest.mark.parametrize("cfg,K,N", [(0, 128, 64), (0, 64, 64), (3, 64, 64), (3, 64, 128), (0, 8, 16),
                                     (4, 64, 64), (4, 64, 128), (4, 8, 16)])
def test_umma_gemm_configs(cfg, K, N):
    e3 = run(cfg, K, N, 1)
    e1 = run(cfg, K, N, 0)
    assert e3 < 2e-6, (cfg, K, N, e3, e1)
    assert e1 < 3e-3, (cfg, K, N, e3, e1)
