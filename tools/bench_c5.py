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
from paper_2205_08115_b200 import instances as I


def problems(batch, seed=0, n=128):
    # Distinct graphs for the first 64 members, then reused (generation is
    # host-bound and the kernel cost does not depend on the graph).
    base = [I.config5_problem(k, seed=seed, n=n) for k in range(min(batch, 64))]
    return [base[k % len(base)] for k in range(batch)]


def run(batch=4096, iters=500, n=128, trace=False):
    probs = problems(batch, n=n)
    cfg = gw.SolverConfig(algorithm="bapg", rho=0.1, max_iters=iters, rel_tol=1e-30, quiet=True)
    args = ([gw.DistanceMatrix.trusted(p.dx) for p in probs],
            [gw.DistanceMatrix.trusted(p.dy) for p in probs],
            [gw.ProbabilityVector(p.mu) for p in probs], [gw.ProbabilityVector(p.nu) for p in probs])
    gw.bapg_solve_batched(*(a[:min(batch, 148)] for a in args), cfg, with_trace=False)  # warm-up
    t0 = time.perf_counter()
    reps = gw.bapg_solve_batched(*args, cfg, with_trace=trace)
    wall = time.perf_counter() - t0
    ms, cnt = C.c_double(), C.c_int64()
    fn = abi.load().gwb_batched_last_kernel_ms
    fn.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    fn(C.byref(ms), C.byref(cnt))
    flops = 2.0 * 2.0 * n * n * (n + n) * batch  # 4 GEMMs of n³ MACs per iteration, all problems
    # Executed tensor work: 128-padded tiles, 3 bf16 planes per GEMM.
    exec_flops = 4 * 3 * 2.0 * 128 ** 3 * batch
    k_s = ms.value * 1e-3
    return {"config": f"c5 {batch} x ER({n},0.1), {iters} it", "kernel_ms": ms.value,
            "problems": cnt.value, "batched_it_per_s": iters / k_s,
            "e2e_batched_it_per_s": iters / wall, "e2e_s": wall,
            "tflops_alg": flops * iters / k_s / 1e12,
            "tflops_exec_bf16": exec_flops * iters / k_s / 1e12,
            "iterations_used": int(reps[0].iterations_used)}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=500)
    ap.add_argument("--size", type=int, default=128)
    a = ap.parse_args()
    print(json.dumps(run(a.batch, a.iters, a.size)), flush=True)
