"""kind::mxf4 operand path: E2M1 0/1 operands with
unit UE8M0 block scales and FP32 accumulation give exact integer dot products.

The probe runs one tcgen05.mma chain D = A B^T (B[i][k] = h[i + k], the
overlapping-window B operand of the extraction kernel) and compares it with an
integer matmul; the largest sums the extraction produces (all-ones inputs at
n = 2^16, K = 65,536 in one accumulator) are covered end to end by
test_gpu_karatsuba.py::test_all_ones[...-65536-45875-2-0] and the dense parity
tests in test_gpu_parity.py.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2011_04130_b200 as q
    from paper_2011_04130_b200 import build
    build.build()
    q.load_library()
    return q


def test_default_build_uses_mxf4(q):
    assert q.gemm_operand_bits() == 4


@pytest.mark.parametrize("K", [64, 256, 1024])
@pytest.mark.parametrize("N", [16, 192, 256])
@pytest.mark.parametrize("data", ["random", "ones", "sparse"])
@pytest.mark.parametrize("hi_first", [False, True])
def test_probe_exact(q, K, N, data, hi_first):
    rng = np.random.default_rng(K * 1000 + N)
    if data == "random":
        A = rng.integers(0, 2, (128, K), dtype=np.uint8)
        h = rng.integers(0, 2, N + K, dtype=np.uint8)
    elif data == "ones":
        A = np.ones((128, K), np.uint8)
        h = np.ones(N + K, np.uint8)
    else:  # one set bit per row of A and a single set seed bit: isolates slot mapping errors
        A = np.zeros((128, K), np.uint8)
        A[np.arange(128), rng.integers(0, K, 128)] = 1
        h = np.zeros(N + K, np.uint8)
        h[rng.integers(0, N + K)] = 1
    B = np.stack([h[i:i + K] for i in range(N)])
    ref = A.astype(np.int64) @ B.T.astype(np.int64)
    D = q.mxf4_probe(torch.from_numpy(A).cuda(), torch.from_numpy(h).cuda(), N, K, hi_first).cpu().numpy()
    assert np.all(D == np.rint(D))
    assert np.array_equal(D.astype(np.int64), ref)
