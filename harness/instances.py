"""Seeded synthetic workloads of BASELINE.json.

Bench / test harness, not product code.  Edge lists come from the C++
generators in ``harness/libgwbinst.so`` (reference RNG and, where the
reference has one, the reference algorithm; built by ``build.py`` with g++,
no CUDA); dense matrices are built here.  The same arrays feed the GPU path
and the CPU oracle.  The product library ``libgwb.so`` holds no generator.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

import os

_I32P = C.POINTER(C.c_int32)
_DP = C.POINTER(C.c_double)
_FP = C.POINTER(C.c_float)

_SIGS = {
    "gwbinst_gen_barabasi_albert": (C.c_int64, [C.c_int32, C.c_int32, C.c_uint64, _I32P, C.c_int64]),
    "gwbinst_gen_erdos_renyi": (C.c_int64, [C.c_int32, C.c_double, C.c_uint64, _I32P, C.c_int64]),
    "gwbinst_gen_sbm_equal": (C.c_int64, [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_uint64,
                                      _I32P, C.c_int64, _I32P]),
    "gwbinst_edge_noise": (C.c_int64, [C.c_int32, _I32P, C.c_int64, C.c_double, C.c_double, C.c_uint64,
                                   _I32P, C.c_int64]),
    "gwbinst_permute_graph": (C.c_int64, [C.c_int32, _I32P, C.c_int64, C.c_uint64, _I32P, _I32P]),
    "gwbinst_gen_gmm3d": (None, [C.c_int32, C.c_int32, C.c_double, C.c_uint64, _DP]),
    "gwbinst_distance_maxnorm_f32": (None, [C.c_int32, _DP, _FP]),
    "gwbinst_jittered_product": (None, [_DP, C.c_int64, _DP, C.c_int64, C.c_double, C.c_uint64,
                                        _DP]),
}

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgwbinst.so")
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            from paper_2205_08115_b200 import build
            build.build_harness()
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_I32P)


def _call_edges(fn, cap_hint: int, *args):
    cap = max(16, cap_hint)
    while True:
        buf = np.empty(2 * cap, dtype=np.int32)
        cnt = fn(*args, _ip(buf), cap)
        if cnt < 0:
            raise ValueError("invalid generator arguments")
        if cnt <= cap:
            return buf[: 2 * cnt].reshape(-1, 2)
        cap = int(cnt)


def barabasi_albert(n: int, m_attach: int, seed: int) -> np.ndarray:
    """gen_barabasi_albert (tasks.cpp:22-65)."""
    return _call_edges(_lib().gwbinst_gen_barabasi_albert, n * m_attach + 64, n, m_attach, seed)


def erdos_renyi(n: int, p: float, seed: int) -> np.ndarray:
    """G(n, p) = gen_gaussian_partition(n, 1, p, 0, seed) (tasks.cpp:67-112)."""
    return _call_edges(_lib().gwbinst_gen_erdos_renyi, int(p * n * n / 2 * 1.2) + 64, n, p, seed)


def sbm_equal(n: int, k: int, p_in: float, p_out: float, seed: int):
    labels = np.empty(n, dtype=np.int32)
    est = int((p_in * n * n / (2 * k) + p_out * n * n / 2) * 1.2) + 64
    lib = _lib()
    cap = est
    while True:
        buf = np.empty(2 * cap, dtype=np.int32)
        cnt = lib.gwbinst_gen_sbm_equal(n, k, p_in, p_out, seed, _ip(buf), cap, _ip(labels))
        if cnt <= cap:
            return buf[: 2 * cnt].reshape(-1, 2), labels
        cap = int(cnt)


def edge_noise(n: int, edges: np.ndarray, q_remove: float, q_add: float, seed: int) -> np.ndarray:
    e = np.ascontiguousarray(edges, dtype=np.int32)
    cnt = e.shape[0]
    return _call_edges(_lib().gwbinst_edge_noise, cnt + int(q_add * cnt) + 16, n, _ip(e), cnt,
                       q_remove, q_add, seed)


def permute_graph(n: int, edges: np.ndarray, seed: int):
    """permute_graph (tasks.cpp:141-154); returns (edges, perm old→new)."""
    e = np.ascontiguousarray(edges, dtype=np.int32)
    out = np.empty_like(e)
    perm = np.empty(n, dtype=np.int32)
    cnt = _lib().gwbinst_permute_graph(n, _ip(e), e.shape[0], seed, _ip(out), _ip(perm))
    return out[:cnt], perm


def adjacency(n: int, edges: np.ndarray, dtype=np.float64) -> np.ndarray:
    """adjacency_distance (tasks.cpp:167-174): symmetric 0/1, zero diagonal."""
    a = np.zeros((n, n), dtype=dtype, order="F")
    if len(edges):
        a[edges[:, 0], edges[:, 1]] = 1
        a[edges[:, 1], edges[:, 0]] = 1
    return a


def gmm_points(n: int, k: int, sigma: float, seed: int) -> np.ndarray:
    xyz = np.empty((n, 3), dtype=np.float64)
    _lib().gwbinst_gen_gmm3d(n, k, sigma, seed, xyz.ctypes.data_as(_DP))
    return xyz


def distance_maxnorm(xyz: np.ndarray) -> np.ndarray:
    n = xyz.shape[0]
    out = np.empty((n, n), dtype=np.float32)
    x = np.ascontiguousarray(xyz, dtype=np.float64)
    _lib().gwbinst_distance_maxnorm_f32(n, x.ctypes.data_as(_DP), out.ctypes.data_as(_FP))
    return np.asfortranarray(out.astype(np.float64))


def jittered_product(mu: np.ndarray, nu: np.ndarray, jitter: float, seed: int) -> np.ndarray:
    """jittered_product (experiment.cpp:41-58): the reference harness's start,
    μνᵀ with a seeded multiplicative jitter, renormalised.  n×m, Fortran order."""
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    nu = np.ascontiguousarray(nu, dtype=np.float64)
    out = np.empty((mu.size, nu.size), dtype=np.float64, order="F")
    _lib().gwbinst_jittered_product(mu.ctypes.data_as(_DP), mu.size, nu.ctypes.data_as(_DP),
                                    nu.size, float(jitter), seed, out.ctypes.data_as(_DP))
    return out


def mix_seed(seed: int, k: int) -> int:
    """Per-instance seed derivation in the spirit of experiment.cpp:28-33."""
    return (seed * 2654435761 + k) & 0xFFFFFFFFFFFFFFFF


@dataclass
class Instance:
    name: str
    dx: np.ndarray          # n×n fp64, Fortran order, symmetric
    dy: np.ndarray          # m×m
    mu: np.ndarray
    nu: np.ndarray
    solver: dict            # SolverConfig overrides
    ground_truth: Optional[np.ndarray] = None
    meta: dict = field(default_factory=dict)

    @property
    def n(self):
        return self.dx.shape[0]

    @property
    def m(self):
        return self.dy.shape[0]


def alignment_instance(source_edges: np.ndarray, n: int, q: float, seed: int, name: str,
                       solver: dict) -> Instance:
    """Source graph vs its noised (remove q|E|, add q|E|) then permuted copy;
    seed streams follow make_alignment_instance (tasks.cpp:156-165)."""
    noisy = edge_noise(n, source_edges, q, q, mix_seed(seed, 1))
    target, perm = permute_graph(n, noisy, mix_seed(seed, 2))
    u = np.full(n, 1.0 / n)
    return Instance(name, adjacency(n, source_edges), adjacency(n, target), u, u.copy(), solver,
                    ground_truth=perm, meta={"edges": int(len(source_edges))})


def config1(seed: int = 0, n: int = 1000) -> Instance:
    """c1: ER(1000, 0.01) vs permuted copy with 5% edge noise; BAPG rho 0.1, 2000 it."""
    e = erdos_renyi(n, 0.01, seed)
    return alignment_instance(e, n, 0.05, seed, f"c1_er{n}",
                              dict(algorithm="bapg", rho=0.1, max_iters=2000, rel_tol=1e-30))


def config2(seed: int = 0, n: int = 2048, m: int = 1536) -> Instance:
    """c2: two 3-D 8-component GMM clouds (sigma 0.1), max-normalised
    Euclidean distances (fp32-exact values); BAPG rho 0.05, 1000 it."""
    dx = distance_maxnorm(gmm_points(n, 8, 0.1, mix_seed(seed, 11)))
    dy = distance_maxnorm(gmm_points(m, 8, 0.1, mix_seed(seed, 12)))
    return Instance(f"c2_gmm{n}x{m}", dx, dy, np.full(n, 1.0 / n), np.full(m, 1.0 / m),
                    dict(algorithm="bapg", rho=0.05, max_iters=1000, rel_tol=1e-30))


def config3(seed: int = 0, n: int = 4000, k: int = 20) -> Instance:
    """c3: SBM(4000, 20 equal blocks, 0.1/0.005) vs the K×K identity target
    (partition_target, tasks.cpp:216-219); mu ∝ degree+1; BAPG rho 0.5, 500 it."""
    e, labels = sbm_equal(n, k, 0.1, 0.005, mix_seed(seed, 21))
    dx = adjacency(n, e)
    deg = dx.sum(axis=0)
    mu = (deg + 1.0) / np.sum(deg + 1.0)
    return Instance(f"c3_sbm{n}_k{k}", dx, np.asfortranarray(np.eye(k)), mu, np.full(k, 1.0 / k),
                    dict(algorithm="bapg", rho=0.5, max_iters=500, rel_tol=1e-30),
                    ground_truth=labels)


def config4(seed: int = 0, n: int = 20000, algorithm: str = "bapg") -> Instance:
    """c4: BA(20000, m=5) vs permuted copy with 2% edge noise; BAPG rho 0.1,
    200 it (hBPG: eps 0.1, step 5, 10 inner sweeps, switch_iters pinned 100)."""
    e = barabasi_albert(n, 5, mix_seed(seed, 41))
    solver = dict(algorithm="bapg", rho=0.1, max_iters=200, rel_tol=1e-30)
    if algorithm == "hbpg":
        solver = dict(algorithm="hbpg", epsilon_reg=0.1, step=5.0, inner_iters=10,
                      inner_tol=1e-9, switch_iters=100, max_iters=200, rel_tol=1e-30)
    return alignment_instance(e, n, 0.02, seed, f"c4_ba{n}", solver)


def config5_problem(k: int, seed: int = 0, n: int = 128) -> Instance:
    """c5 member k: ER(128, 0.1) vs permuted copy with 5% edge noise."""
    s = mix_seed(seed, 5000 + k)
    e = erdos_renyi(n, 0.1, s)
    return alignment_instance(e, n, 0.05, s, f"c5_er{n}_{k}",
                              dict(algorithm="bapg", rho=0.1, max_iters=500, rel_tol=1e-30))
