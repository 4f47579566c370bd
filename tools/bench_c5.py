"""Config 5 throughput: `batch` independent ER(128, 0.1) alignment problems,
500 BAPG iterations each, through gwb_bapg_solve_batched (on-chip kernel).

Reports batched it/s (= iterations ÷ kernel time, every problem advancing one
iteration per batched iteration), the kernel's algorithmic tensor rate and
the end-to-end rate of the C-ABI call (host fp64 in/out).
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2205_08115_b200 as gw
from paper_2205_08115_b200 import abi
from harness import instances as I


def problems(batch, seed=0, n=128, start=0):
    """`batch` distinct c5 members start, start+1, … (ER(n, 0.1) vs its noised
    permuted copy, per-problem seeds), ~0.5 ms each to generate."""
    return [I.config5_problem(k, seed=seed, n=n) for k in range(start, start + batch)]


def _pinned(count):
    import torch
    return torch.empty(count, dtype=torch.float64, pin_memory=True).numpy()


def run(batch=4096, iters=500, n=128, trace=False, start=0):
    """One gwb_bapg_solve_batched call over `batch` problems: inputs staged in
    pinned host memory beforehand (fp64 column-major, as the C-ABI takes
    them); the timed call includes their H2D copy, the solve and the D2H of
    every final coupling."""
    probs = problems(batch, n=n, start=start)
    cfg = gw.SolverConfig(algorithm="bapg", rho=0.1, max_iters=iters, rel_tol=1e-30,
                          quiet=True).to_abi()
    nn = n * n
    dx, dy = _pinned(batch * nn), _pinned(batch * nn)
    mu, nu = _pinned(batch * n), _pinned(batch * n)
    for k, p in enumerate(probs):
        dx[k * nn:(k + 1) * nn] = np.asarray(p.dx, dtype=np.float64).ravel(order="F")
        dy[k * nn:(k + 1) * nn] = np.asarray(p.dy, dtype=np.float64).ravel(order="F")
        mu[k * n:(k + 1) * n] = p.mu
        nu[k * n:(k + 1) * n] = p.nu
    out = _pinned(batch * nn)
    conv = np.zeros(batch, dtype=np.int32)
    used = np.zeros(batch, dtype=np.int32)
    lib = abi.load()
    D = C.POINTER(C.c_double)
    I32 = C.POINTER(C.c_int32)

    def call(b):
        st = abi.Status()
        lib.gwb_bapg_solve_batched(C.byref(cfg), b, dx.ctypes.data_as(D), n, dy.ctypes.data_as(D),
                                   n, mu.ctypes.data_as(D), nu.ctypes.data_as(D),
                                   out.ctypes.data_as(D), None, None, None, 0, None,
                                   conv.ctypes.data_as(I32), used.ctypes.data_as(I32),
                                   C.byref(st))
        abi.raise_for(st)

    call(batch)  # warm-up step (module load; the stream-ordered pool grows to the batch's size)
    t0 = time.perf_counter()
    call(batch)
    wall = time.perf_counter() - t0
    ms, cnt = C.c_double(), C.c_int64()
    fn = lib.gwb_batched_last_kernel_ms
    fn.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    fn(C.byref(ms), C.byref(cnt))
    flops = 2.0 * 2.0 * n * n * (n + n) * batch  # 4 GEMMs of n³ MACs per iteration, all problems
    # Executed tensor work: 128-padded tiles, 2 fp16 planes per GEMM (f16x2).
    exec_flops = 4 * 2 * 2.0 * 128 ** 3 * batch
    k_s = ms.value * 1e-3
    # Problems stop where rel_change crosses rel_tol (the reference's rule):
    # a batched iteration advances every problem once, so the executed count
    # is the mean iterations used.
    mean_used = float(used.mean())
    return {"config": f"c5 {batch} x ER({n},0.1), {iters} it", "kernel_ms": ms.value,
            "problems": cnt.value, "batched_it_per_s": mean_used / k_s,
            "mean_iterations_used": mean_used,
            "e2e_batched_it_per_s": mean_used / wall, "e2e_s": wall,
            "h2d_bytes": int(dx.nbytes + dy.nbytes + mu.nbytes + nu.nbytes),
            "d2h_bytes": int(out.nbytes),
            "tflops_alg": flops * mean_used / k_s / 1e12,
            "tflops_exec_f16": exec_flops * mean_used / k_s / 1e12,
            "iterations_used": int(used.min()), "iterations_used_max": int(used.max()),
            "converged_any": bool(conv.any()),
            "final_sum_err": float(np.abs(out.reshape(batch, -1).sum(axis=1) - 1.0).max())}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=500)
    ap.add_argument("--size", type=int, default=128)
    a = ap.parse_args()
    print(json.dumps(run(a.batch, a.iters, a.size)), flush=True)
