"""Diagnostic: accumulation error of the split-operand tensor-core GEMM on
all-positive operands (c2's distances and couplings) vs the same product
formed from centred operands plus exact rank-1 terms:

    A·Bᵀ = (A0 + a)(B0 + b)ᵀ = A0·B0ᵀ + b·rowsum(A) 1ᵀ + a·1 colsum... (fp64)

    python tools/center_probe.py [K]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from tests.test_gpu_gemm import _gemm  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    rng = np.random.default_rng(9)
    M = N = 512
    a = rng.uniform(0.0, 1.0, (M, K)).astype(np.float32)
    b = rng.uniform(0.0, 1.0, (N, K)).astype(np.float32) * np.float32(1e-3)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    for prec, name in ((8, "f16x3"), (2, "3xtf32")):
        c = _gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), prec)
        e = (c - ref) / ref
        line = f"{name} K={K}: plain mean {e.mean():.2e} max {np.abs(e).max():.2e}"
        # centre A only (the structure matrix): A0 = A - ca, exact-ish in fp32
        for ca in (0.5, float(a.mean())):
            a0 = (a.astype(np.float64) - ca).astype(np.float32)
            c0 = _gemm(torch.from_numpy(a0).cuda(), torch.from_numpy(b).cuda(), prec)
            corr = ca * b.astype(np.float64).sum(axis=1)[None, :]
            full = c0 + corr + (a0.astype(np.float64) + ca - a.astype(np.float64)) @ b.astype(np.float64).T
            e0 = (full - ref) / ref
            line += f" | centre {ca:.3f}: mean {e0.mean():.2e} max {np.abs(e0).max():.2e}"
        print(line, flush=True)


if __name__ == "__main__":
    main()
