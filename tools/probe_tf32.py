"""Probe how tcgen05.mma kind::tf32 converts fp32 operands and accumulates."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from tests.test_gpu_gemm import _gemm

def run(a, b, prec):
    return _gemm(torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda(),
                 torch.from_numpy(np.ascontiguousarray(b, np.float32)).cuda(), prec)

M, N, K = 128, 256, 32
# 1) conversion: a = 1 + f*2^-10 for fractional f, b = 1 (one nonzero k)
fr = np.array([0.0, 0.25, 0.49, 0.5, 0.51, 0.75, 0.99])
a = np.zeros((M, K), np.float32); b = np.zeros((N, K), np.float32)
for i, f in enumerate(fr):
    a[i, 0] = np.float32(1.0 + f * 2.0**-10)
b[:, 0] = 1.0
c = run(a, b, 1)
for i, f in enumerate(fr):
    print(f"conv a=1+{f}*2^-10 -> (c-1)/2^-10 = {(c[i,0]-1)/2**-10:.4f}")
# 2) accumulation: K terms that are exact in tf32; exact sum needs 24+ bits
K2 = 1024
a = np.zeros((M, K2), np.float32); b = np.zeros((N, K2), np.float32)
a[0, 0] = 2.0**12; a[0, 1:] = 2.0**-11   # big + many small
b[:, :] = 1.0
c = run(a, b, 1)
exact = 2.0**12 + (K2 - 1) * 2.0**-11
print(f"accum: got {c[0,0]!r} exact {exact!r} fp32(exact) {np.float32(exact)!r} err_ulps {(c[0,0]-exact)/np.spacing(np.float32(4096)):.2f}")
a[0, 0] = 1.0; a[0, 1:] = 2.0**-24 * 3
c = run(a, b, 1); exact = 1.0 + (K2-1)*3*2.0**-24
print(f"accum small: got {c[0,0]!r} exact {exact!r}")
# 3) random 3x error vs K
rng = np.random.default_rng(1)
for K3 in (32, 256, 1024):
    a = rng.random((384, K3)).astype(np.float32); b = rng.random((640, K3)).astype(np.float32)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    for p in (1, 2):
        c = run(a, b, p)
        print(f"K={K3} prec={p} rel={np.abs(c-ref).max()/np.abs(ref).max():.3e} mean={np.mean(c-ref)/np.mean(ref):.3e}")
