"""K1: the tcgen05 TF32 / 3xTF32 GEMM against an fp64 torch reference."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gemm(a, b, precision, c=None):
    import torch
    from paper_2205_08115_b200 import abi
    M, K = a.shape
    N = b.shape[0]
    ld = lambda k: (k + 31) // 32 * 32
    A = torch.zeros((M, ld(K)), device="cuda", dtype=torch.float32); A[:, :K] = a
    B = torch.zeros((N, ld(K)), device="cuda", dtype=torch.float32); B[:, :K] = b
    Cm = torch.full((M, ld(N)), float("nan"), device="cuda", dtype=torch.float32)
    lib = abi.load()
    fn = lib.gwb_debug_gemm
    fn.restype = C.c_int32
    fn.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                   C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_void_p, C.POINTER(abi.Status)]
    st = abi.Status()
    torch.cuda.synchronize()
    rc = fn(A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], Cm.data_ptr(), Cm.shape[1],
            M, N, K, precision, None, C.byref(st))
    torch.cuda.synchronize()
    assert rc == 0, st.message
    return Cm[:, :N].double().cpu().numpy()


# (1536, 2048, 512) and (1500, 1900, 300) select 192-wide tiles (gemm_plan_create:
# 48 tiles of 256 vs 60-66 of 192 on 74 SM pairs), the ragged one with a
# partial last tile; (1000, 1000, 1000) selects 128-wide tiles with split-K;
# (5000, 5000, 64) and (4500, 4700, 96) keep 256-wide tiles (> 4 waves), whose
# epilogue writes rows by bulk copies — the ragged one also takes the direct
# store path on its partial last column tile.
@pytest.mark.parametrize("M,N,K", [(128, 256, 32), (256, 512, 256), (1000, 1000, 1000),
                                   (200, 72, 40), (20, 4000, 20), (4000, 20, 4000),
                                   (1536, 2048, 512), (1500, 1900, 300),
                                   (5000, 5000, 64), (4500, 4700, 96)])
def test_gemm_tf32_exact_operands(gpu, M, N, K):
    # Integer-valued operands are exact in TF32 and sums stay < 2^24: the
    # tensor-core result must be bit-exact.
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    a = rng.integers(0, 3, size=(M, K)).astype(np.float32)
    b = rng.integers(0, 3, size=(N, K)).astype(np.float32)
    import torch
    c = _gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), 1)
    np.testing.assert_array_equal(c, a.astype(np.float64) @ b.astype(np.float64).T)


@pytest.mark.parametrize("precision,tol", [(1, 2e-3), (2, 2e-6), (8, 1e-6)])
def test_gemm_precision(gpu, precision, tol):
    import torch
    rng = np.random.default_rng(1)
    M, N, K = 384, 640, 1024
    a = rng.random((M, K)).astype(np.float32)
    b = rng.random((N, K)).astype(np.float32)
    c = _gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), precision)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    rel = np.abs(c - ref).max() / np.abs(ref).max()
    assert rel < tol, rel


@pytest.mark.parametrize("precision", [7, 3])  # f16x2, bf16x3 split-plane chains
def test_split_gemm_long_k_accumulation(gpu, precision):
    # c4-length K with all-positive terms (the worst case for the tensor
    # core's truncating accumulation): 0/1 A × positive B against fp64.
    # The promotion of each chunk into fp32 registers bounds the bias.
    import torch
    rng = np.random.default_rng(3)
    M, N, K = 256, 256, 20000
    a = (rng.random((M, K)) < 0.5).astype(np.float32)
    b = rng.uniform(0.25, 1.0, (N, K)).astype(np.float32)
    c = _gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), precision)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    err = (c - ref) / ref
    assert np.abs(err).max() < 2e-6, (np.abs(err).max(), err.mean())


@pytest.mark.parametrize("precision", [2, 8])  # 3xTF32, f16x3 (weighted operands)
def test_weighted_gemm_bias(gpu, precision):
    """Both operands weighted (c2's Euclidean distances): the mean relative
    error measures the chain's accumulation bias, the max its noise.  kind::f16
    (f16x3) must be at least 5x less biased than kind::tf32 (3xTF32)."""
    import torch
    rng = np.random.default_rng(9)
    M, N, K = 512, 512, 2048
    a = rng.uniform(0.0, 1.0, (M, K)).astype(np.float32)
    b = rng.uniform(0.0, 1.0, (N, K)).astype(np.float32)
    c = _gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), precision)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    err = (c - ref) / ref
    print(f"precision {precision}: mean rel err {err.mean():.2e}, max {np.abs(err).max():.2e}")
    if precision == 8:
        assert abs(err.mean()) < 6e-7 and np.abs(err).max() < 1.5e-6
    else:
        assert np.abs(err).max() < 5e-6
