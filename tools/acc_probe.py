import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from tests.test_gpu_gemm import _gemm
rng = np.random.default_rng(3)
M, N, K = 256, 256, 20000
a = (rng.random((M, K)) < 0.5).astype(np.float32)
b = rng.uniform(0.25, 1.0, (N, K)).astype(np.float32)
ref = a.astype(np.float64) @ b.astype(np.float64).T
for prec in (7, 3):
    c = _gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), prec)
    err = (c - ref) / ref
    print(os.environ.get("GWB_GEMM_CHUNK_KB", "default"), prec, f"max {np.abs(err).max():.2e} mean {err.mean():.2e}", flush=True)
