"""16-bit tcgen05 bring-up: kind::f16 (BF16 in, F32 accumulate) with bf16x3-split operands in
the 16-bit CM layout, every K-major / MN-major combination, M = 64 and 128, vs float64."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2308_02494_b200 import _lib as L  # noqa: E402


def run(mode, M, K, N, split3, seed=0):
    rng = np.random.default_rng(seed + 7 * mode + M + K + N)
    A = rng.normal(size=(M, K)).astype(np.float32)
    B = rng.normal(size=(K, N)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    d = L.zeros((M, N), np.float32)
    a_d, b_d = L.to_device(A), L.to_device(B)
    L.check(L.debug_lib().apmg_debug_umma_bf16(mode, M, K, N, split3, L.ptr(a_d), L.ptr(b_d), L.ptr(d),
                                         L.stream_handle()), "umma_bf16")
    got = L.to_host(d).astype(np.float64)
    return float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
@pytest.mark.parametrize("M,K,N", [(64, 64, 64), (128, 128, 64), (128, 64, 128), (64, 16, 16)])
def test_bf16x3_gemm(mode, M, K, N):
    e6 = run(mode, M, K, N, 1)
    e1 = run(mode, M, K, N, 0)
    assert e6 < 2e-6, (mode, M, K, N, e6, e1)
    assert e1 < 2e-2, (mode, M, K, N, e6, e1)
