"""Python mirror of the reference solver interface (``gw::`` namespace).

Names, argument meaning, validation order and exception classes follow
``/root/reference/proj/include/gw/{types,solvers,projections,diagnostics}.hpp``
so parity tests read like the reference's own tests.  Every compute call goes
through the C-ABI in ``libgwb.so`` (include/gwb.h); there is no Python or CPU
fallback for the solver path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import abi
from .abi import (ConfigError, DimensionMismatchError, NumericalInstabilityError,  # noqa: F401
                  UnsupportedError, ZeroSumLineError, DomainError)

ROWS, COLS = abi.ROWS, abi.COLS


def _f64(a, order="F") -> np.ndarray:
    return np.require(np.asarray(a, dtype=np.float64), requirements=[order[0] + "_CONTIGUOUS", "ALIGNED"])


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ---------------------------------------------------------------------------
# Value types (types.hpp:62-118, types.cpp:68-153)
# ---------------------------------------------------------------------------
class DistanceMatrix:
    """Symmetric nonnegative structure matrix; construction symmetrizes
    (A + Aᵀ)/2 and rejects negative or non-finite entries (types.cpp:68-84)."""

    def __init__(self, entries):
        a = np.asarray(entries, dtype=np.float64)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            r, c = (a.shape + (0, 0))[:2] if a.ndim == 2 else (a.size, 1)
            raise DimensionMismatchError(f"distance matrix must be square, got {r}x{c}")
        if a.shape[0] == 0:
            raise DimensionMismatchError("distance matrix must be nonempty")
        e = 0.5 * (a + a.T)
        if not np.all(np.isfinite(e)):
            raise ValueError("distance matrix has non-finite entries")
        if np.any(e < 0.0):
            raise ValueError("distance matrix has negative entries")
        self._e = np.asfortranarray(e)

    @classmethod
    def trusted(cls, entries: np.ndarray) -> "DistanceMatrix":
        """Wrap an already-symmetric, validated matrix without the O(n²) copy."""
        obj = cls.__new__(cls)
        obj._e = _f64(entries)
        return obj

    def size(self) -> int:
        g = getattr(self, "_graph", None)
        return g.num_nodes() if g is not None else self._e.shape[0]

    def entries(self) -> np.ndarray:
        if getattr(self, "_e", None) is None:  # graph-backed: materialise on demand
            g = self._graph
            a = np.zeros((g.num_nodes(), g.num_nodes()), order="F")
            e = g.edges()
            a[e[:, 0], e[:, 1]] = 1.0
            a[e[:, 1], e[:, 0]] = 1.0
            self._e = a
        return self._e

    def graph(self) -> Optional["Graph"]:
        """The Graph this matrix is the adjacency of (adjacency_distance), or None."""
        return getattr(self, "_graph", None)


class Graph:
    """gw::Graph (types.hpp:120-130, types.cpp:155-174): edges stored as
    canonical (min, max) pairs, sorted, duplicates removed."""

    def __init__(self, num_nodes: int, edges):
        if num_nodes <= 0:
            raise ValueError("graph must have at least one node")
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        for a, b in e:
            if a == b:
                raise ValueError(f"self-loop at node {a}")
            if a < 0 or b < 0 or a >= num_nodes or b >= num_nodes:
                raise ValueError(f"edge ({a},{b}) out of range for {num_nodes} nodes")
        canon = np.stack([e.min(axis=1), e.max(axis=1)], axis=1) if len(e) else e
        self._n = int(num_nodes)
        self._edges = np.unique(canon, axis=0).astype(np.int32) if len(e) else \
            np.zeros((0, 2), dtype=np.int32)

    def num_nodes(self) -> int:
        return self._n

    def edges(self) -> np.ndarray:
        return self._edges


def adjacency_distance(g: Graph) -> DistanceMatrix:
    """gw::adjacency_distance (tasks.cpp:167-174): the 0/1 adjacency.  The
    matrix keeps its graph, so `solve` builds it on the device from the edge
    list (gwb_solve_graphs) instead of uploading n² fp64 entries."""
    dm = DistanceMatrix.__new__(DistanceMatrix)
    dm._e = None
    dm._graph = g
    return dm


class ProbabilityVector:
    """Strictly positive weights summing to 1 within 1e-12 (types.cpp:86-108)."""

    def __init__(self, weights):
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64).ravel())
        if w.size == 0:
            raise ValueError("probability vector must be nonempty")
        if not np.all(np.isfinite(w)):
            raise ValueError("probability vector has non-finite entries")
        if np.any(w <= 0.0):
            raise ValueError("probability vector entries must be strictly positive; remove "
                             "zero-mass points before construction")
        mass = float(np.sum(w))
        if abs(mass - 1.0) > 1e-12:
            raise ValueError(f"probability vector sums to {mass:g}, expected 1 within 1e-12")
        self._w = w

    @staticmethod
    def uniform(n: int) -> "ProbabilityVector":
        return ProbabilityVector(np.full(n, 1.0 / n))

    def size(self) -> int:
        return self._w.size

    def weights(self) -> np.ndarray:
        return self._w


class Coupling:
    """Nonnegative matrix of total mass 1 within 1e-9 (types.cpp:110-126)."""

    def __init__(self, entries):
        e = np.asarray(entries, dtype=np.float64)
        if e.ndim != 2 or e.shape[0] == 0 or e.shape[1] == 0:
            raise DimensionMismatchError("coupling must be nonempty")
        if not np.all(np.isfinite(e)):
            raise ValueError("coupling has non-finite entries")
        if np.any(e < 0.0):
            raise ValueError("coupling has negative entries")
        mass = float(np.sum(e))
        if abs(mass - 1.0) > 1e-9:
            raise ValueError(f"coupling total mass is {mass:g}, expected 1 within 1e-9")
        self._e = e

    def rows(self) -> int:
        return self._e.shape[0]

    def cols(self) -> int:
        return self._e.shape[1]

    def entries(self) -> np.ndarray:
        return self._e


@dataclass
class SolverConfig:
    """gw::SolverConfig with the protocol defaults (types.hpp:132-147)."""

    algorithm: str = "bapg"
    geometry: str = "entropy"
    rho: float = 0.1
    step: float = 5.0
    epsilon_reg: float = 0.1
    inner_iters: int = 1000
    inner_tol: float = 1e-9
    rel_tol: float = 1e-6
    max_iters: int = 2000
    perturbation: float = 0.0
    switch_iters: int = 200
    seed: int = 0
    log_domain: bool = False
    record_residual: bool = False
    # B200 extensions
    precision: str = "auto"   # auto | tf32 | 3xtf32 | bf16x3 | bf16x2 | f16x2 | f16x3 | sparse | fp32
    quiet: bool = False

    def to_abi(self) -> abi.Config:
        prec = {"auto": abi.PREC_AUTO, "tf32": abi.PREC_TF32, "3xtf32": abi.PREC_3XTF32,
                "bf16x3": abi.PREC_BF16X3, "bf16x2": abi.PREC_BF16X2,
                "sparse": abi.PREC_SPARSE, "fp32": abi.PREC_FP32,
                "f16x2": abi.PREC_F16X2, "f16x3": abi.PREC_F16X3}
        if self.algorithm not in abi.ALGORITHMS:
            raise ConfigError(f"unknown solver '{self.algorithm}' (expected bapg|bpg|ebpg|hbpg|fw)")
        if self.geometry not in ("entropy", "quadratic"):
            raise ConfigError(f"unknown geometry '{self.geometry}' (expected entropy|quadratic)")
        return abi.default_config(
            algorithm=abi.ALGORITHMS[self.algorithm],
            geometry=abi.ENTROPY if self.geometry == "entropy" else abi.QUADRATIC,
            rho=self.rho, step=self.step, epsilon_reg=self.epsilon_reg,
            inner_iters=self.inner_iters, inner_tol=self.inner_tol, rel_tol=self.rel_tol,
            max_iters=self.max_iters, perturbation=self.perturbation,
            switch_iters=self.switch_iters, seed=self.seed, log_domain=int(self.log_domain),
            record_residual=int(self.record_residual), precision=prec[self.precision],
            quiet=int(self.quiet))


def validate(config: SolverConfig) -> None:
    """gw::validate (types.cpp:176-188)."""
    st = abi.Status()
    abi.load().gwb_validate_config(C.byref(config.to_abi()), C.byref(st))
    abi.raise_for(st)


def validate_inputs(d_x: DistanceMatrix, d_y: DistanceMatrix, mu: ProbabilityVector,
                    nu: ProbabilityVector) -> None:
    """gw::validate_inputs (types.cpp:190-202)."""
    if d_x.size() != mu.size():
        raise DimensionMismatchError(
            f"D_X is {d_x.size()}x{d_x.size()} but mu has length {mu.size()}")
    if d_y.size() != nu.size():
        raise DimensionMismatchError(
            f"D_Y is {d_y.size()}x{d_y.size()} but nu has length {nu.size()}")


@dataclass
class IterationRecord:
    iter: int = 0
    objective: float = 0.0
    marginal_infeasibility: float = 0.0
    split_gap: float = 0.0
    residual: Optional[float] = None
    rel_change: float = 0.0
    elapsed_seconds: float = 0.0
    phase: int = 0


@dataclass
class SolveReport:
    final_coupling: Coupling
    pi_half: Optional[Coupling] = None
    w_half: Optional[Coupling] = None
    trace: List[IterationRecord] = field(default_factory=list)
    converged: bool = False
    iterations_used: int = 0


@dataclass
class SolveOptions:
    initial: Optional[np.ndarray] = None
    observer: Optional[Callable[[int, np.ndarray, Optional[np.ndarray]], None]] = None


_ENTRY = {None: "gwb_solve", "bapg": "gwb_bapg_solve", "bpg": "gwb_bpg_solve",
          "ebpg": "gwb_ebpg_solve", "hbpg": "gwb_hbpg_solve"}


def _solve(entry, d_x, d_y, mu, nu, config, opts):
    lib = abi.load()
    opts = opts or SolveOptions()
    cfg = config.to_abi()
    # Validation order of the reference (solvers.cpp:141-143): the algorithm
    # and config checks run in the C-ABI; dimension checks need the objects.
    if entry is not None and cfg.algorithm != abi.ALGORITHMS[entry]:
        raise ConfigError(f"{entry}_solve called with algorithm '{config.algorithm}'")
    validate(config)
    validate_inputs(d_x, d_y, mu, nu)
    n, m = d_x.size(), d_y.size()
    init = None
    if opts.initial is not None:
        init = _f64(opts.initial)
        if init.shape != (n, m):
            raise DimensionMismatchError("initial coupling shape mismatch")
    out_final = np.empty((n, m), dtype=np.float64, order="F")
    is_bapg = cfg.algorithm == abi.BAPG
    out_pi = np.empty((n, m), dtype=np.float64, order="F") if is_bapg else None
    out_w = np.empty((n, m), dtype=np.float64, order="F") if is_bapg else None
    cap = max(1, config.max_iters)
    trace = (abi.Record * cap)()
    n_rec, conv, used = C.c_int32(0), C.c_int32(0), C.c_int32(0)
    st = abi.Status()

    cb = abi.OBSERVER()
    raised = []
    if opts.observer is not None:
        def _obs(_user, it, pi_p, w_p, nn, mm):
            # An exception in the observer aborts the solve and reaches the
            # caller unchanged, as a C++ observer's would (solvers.cpp:206).
            try:
                pi = np.ctypeslib.as_array(pi_p, shape=(nn * mm,)).reshape((nn, mm), order="F").copy()
                w = None
                if w_p:
                    w = np.ctypeslib.as_array(w_p, shape=(nn * mm,)).reshape((nn, mm), order="F").copy()
                opts.observer(int(it), pi, w)
                return 0
            except BaseException as ex:  # noqa: BLE001 — rethrown after the call
                raised.append(ex)
                return 1
        cb = abi.OBSERVER(_obs)
    gx, gy = d_x.graph(), d_y.graph()
    if gx is not None and gy is not None:
        # Both are adjacency_distance(graph): D is built on the device.
        ex, ey = np.ascontiguousarray(gx.edges()), np.ascontiguousarray(gy.edges())
        i32 = C.POINTER(C.c_int32)
        lib.gwb_solve_graphs(C.byref(cfg), n, ex.ctypes.data_as(i32), len(ex), m,
                             ey.ctypes.data_as(i32), len(ey), _ptr(mu.weights()),
                             _ptr(nu.weights()), _ptr(init), cb, None, _ptr(out_final),
                             _ptr(out_pi), _ptr(out_w), trace, cap, C.byref(n_rec),
                             C.byref(conv), C.byref(used), C.byref(st))
    else:
        fn = getattr(lib, _ENTRY[entry])
        fn(C.byref(cfg), _ptr(d_x.entries()), n, _ptr(d_y.entries()), m, _ptr(mu.weights()),
           _ptr(nu.weights()), _ptr(init), cb, None, _ptr(out_final), _ptr(out_pi),
           _ptr(out_w), trace, cap, C.byref(n_rec), C.byref(conv), C.byref(used), C.byref(st))
    if raised:
        raise raised[0]
    abi.raise_for(st)
    recs = [IterationRecord(iter=r.iter, objective=r.objective,
                            marginal_infeasibility=r.marginal_infeasibility,
                            split_gap=r.split_gap,
                            residual=r.residual if r.has_residual else None,
                            rel_change=r.rel_change, elapsed_seconds=r.elapsed_seconds,
                            phase=r.phase) for r in trace[: n_rec.value]]
    return SolveReport(final_coupling=Coupling(out_final),
                       pi_half=Coupling(out_pi) if is_bapg else None,
                       w_half=Coupling(out_w) if is_bapg else None,
                       trace=recs, converged=bool(conv.value), iterations_used=used.value)


def solve(d_x, d_y, mu, nu, config: SolverConfig, opts: Optional[SolveOptions] = None):
    """gw::solve (solvers.cpp:499-515)."""
    return _solve(None, d_x, d_y, mu, nu, config, opts)


def bapg_solve(d_x, d_y, mu, nu, config: SolverConfig, opts=None):
    """gw::bapg_solve (solvers.cpp:138-217)."""
    return _solve("bapg", d_x, d_y, mu, nu, config, opts)


def bapg_solve_batched(d_xs, d_ys, mus, nus, config: SolverConfig,
                       with_trace: bool = True) -> List[SolveReport]:
    """Batched BAPG over independent problems of one shape (config 5).

    Equivalent to ``[bapg_solve(dx, dy, mu, nu, config) for ...]`` — the
    reference's experiment worker pool (experiment.cpp:273-304) — but solved
    by the on-chip batched kernel (n, m ≤ 128) in one device call.  The first
    failing problem (lowest index) raises, its index named in the message.
    """
    lib = abi.load()
    cfg = config.to_abi()
    if cfg.algorithm != abi.BAPG:
        raise ConfigError(f"bapg_solve called with algorithm '{config.algorithm}'")
    validate(config)
    batch = len(d_xs)
    if batch == 0 or not (len(d_ys) == len(mus) == len(nus) == batch):
        raise DimensionMismatchError("batched inputs must be nonempty and of equal length")
    for args in zip(d_xs, d_ys, mus, nus):
        validate_inputs(*args)
    n, m = d_xs[0].size(), d_ys[0].size()
    if any(d.size() != n for d in d_xs) or any(d.size() != m for d in d_ys):
        raise DimensionMismatchError("batched problems must share n and m")
    dx = np.concatenate([_f64(d.entries()).ravel(order="F") for d in d_xs])
    dy = np.concatenate([_f64(d.entries()).ravel(order="F") for d in d_ys])
    mu = np.concatenate([np.asarray(p.weights(), dtype=np.float64) for p in mus])
    nu = np.concatenate([np.asarray(p.weights(), dtype=np.float64) for p in nus])
    out_final = np.empty(batch * n * m)
    out_pi = np.empty(batch * n * m)
    out_w = np.empty(batch * n * m)
    cap = max(1, config.max_iters) if with_trace else 0
    trace = (abi.Record * (batch * cap))() if with_trace else None
    n_rec = np.zeros(batch, dtype=np.int32)
    conv = np.zeros(batch, dtype=np.int32)
    used = np.zeros(batch, dtype=np.int32)
    st = abi.Status()
    lib.gwb_bapg_solve_batched(C.byref(cfg), batch, _ptr(dx), n, _ptr(dy), m, _ptr(mu), _ptr(nu),
                               _ptr(out_final), _ptr(out_pi), _ptr(out_w), trace, cap,
                               n_rec.ctypes.data_as(C.POINTER(C.c_int32)),
                               conv.ctypes.data_as(C.POINTER(C.c_int32)),
                               used.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(st))
    abi.raise_for(st)
    out = []
    for b in range(batch):
        sl = slice(b * n * m, (b + 1) * n * m)
        recs = []
        if with_trace:
            recs = [IterationRecord(iter=r.iter, objective=r.objective,
                                    marginal_infeasibility=r.marginal_infeasibility,
                                    split_gap=r.split_gap, rel_change=r.rel_change,
                                    elapsed_seconds=r.elapsed_seconds, phase=r.phase,
                                    residual=r.residual if r.has_residual else None)
                    for r in trace[b * cap: b * cap + int(n_rec[b])]]
        shape = lambda a: Coupling(a[sl].reshape((n, m), order="F"))
        out.append(SolveReport(final_coupling=shape(out_final), pi_half=shape(out_pi),
                               w_half=shape(out_w), trace=recs, converged=bool(conv[b]),
                               iterations_used=int(used[b])))
    return out


def bpg_solve(d_x, d_y, mu, nu, config: SolverConfig, opts=None):
    """gw::bpg_solve (solvers.cpp:219-293)."""
    return _solve("bpg", d_x, d_y, mu, nu, config, opts)


def ebpg_solve(d_x, d_y, mu, nu, config: SolverConfig, opts=None):
    """gw::ebpg_solve (solvers.cpp:295-363)."""
    return _solve("ebpg", d_x, d_y, mu, nu, config, opts)


def hbpg_solve(d_x, d_y, mu, nu, config: SolverConfig, opts=None):
    """gw::hbpg_solve (solvers.cpp:365-426)."""
    return _solve("hbpg", d_x, d_y, mu, nu, config, opts)


def gw_objective(d_x: DistanceMatrix, d_y: DistanceMatrix, pi) -> float:
    """gw::gw_objective (solvers.cpp:64-69)."""
    p = _f64(pi)
    out = C.c_double(0.0)
    st = abi.Status()
    abi.load().gwb_gw_objective(_ptr(d_x.entries()), d_x.size(), _ptr(d_y.entries()), d_y.size(),
                                _ptr(p), p.shape[0], p.shape[1], C.byref(out), C.byref(st))
    abi.raise_for(st)
    return out.value


def product_coupling(mu: ProbabilityVector, nu: ProbabilityVector) -> Coupling:
    """gw::product_coupling (types.cpp:204-207)."""
    out = np.empty((mu.size(), nu.size()), order="F")
    st = abi.Status()
    abi.load().gwb_product_coupling(_ptr(mu.weights()), mu.size(), _ptr(nu.weights()), nu.size(),
                                    _ptr(out), C.byref(st))
    abi.raise_for(st)
    return Coupling(out)


def lipschitz_bound(d_x: DistanceMatrix, d_y: DistanceMatrix) -> float:
    """gw::lipschitz_bound (solvers.cpp:133-136)."""
    out = C.c_double(0.0)
    st = abi.Status()
    abi.load().gwb_lipschitz_bound(_ptr(d_x.entries()), d_x.size(), _ptr(d_y.entries()),
                                   d_y.size(), C.byref(out), C.byref(st))
    abi.raise_for(st)
    return out.value


def kl_scale(pi, target: ProbabilityVector, axis: int) -> np.ndarray:
    """gw::kl_scale (projections.cpp:12-34)."""
    p = _f64(pi)
    out = np.empty_like(p, order="F")
    st = abi.Status()
    abi.load().gwb_kl_scale(_ptr(p), p.shape[0], p.shape[1], _ptr(target.weights()),
                            target.size(), axis, _ptr(out), C.byref(st))
    abi.raise_for(st)
    return out


@dataclass
class SinkhornResult:
    coupling: np.ndarray
    iterations: int = 0
    marginal_error: float = 0.0
    converged: bool = False


def _sinkhorn(k, mu, nu, tol, max_iters, log_domain):
    a = _f64(k)
    n, m = a.shape
    if n != mu.size() or m != nu.size():
        name = "sinkhorn_project_log: exponent/marginal" if log_domain else "sinkhorn_project: kernel/marginal"
        raise DimensionMismatchError(f"{name} shape mismatch")
    out = np.empty_like(a, order="F")
    it, err, conv = C.c_int32(0), C.c_double(0.0), C.c_int32(0)
    st = abi.Status()
    abi.load().gwb_sinkhorn_project(_ptr(a), n, m, _ptr(mu.weights()), _ptr(nu.weights()), tol,
                                    max_iters, int(log_domain), _ptr(out), C.byref(it),
                                    C.byref(err), C.byref(conv), C.byref(st))
    abi.raise_for(st)
    return SinkhornResult(out, it.value, err.value, bool(conv.value))


def sinkhorn_project(kernel, mu, nu, tol, max_iters) -> SinkhornResult:
    """gw::sinkhorn_project (projections.cpp:92-116)."""
    return _sinkhorn(kernel, mu, nu, tol, max_iters, False)


def sinkhorn_project_log(exponent, mu, nu, tol, max_iters) -> SinkhornResult:
    """gw::sinkhorn_project_log (projections.cpp:129-163)."""
    return _sinkhorn(exponent, mu, nu, tol, max_iters, True)


def marginal_infeasibility(pi, mu: ProbabilityVector, nu: ProbabilityVector) -> float:
    """gw::marginal_infeasibility (diagnostics.cpp:9-20)."""
    p = _f64(pi)
    out = C.c_double(0.0)
    st = abi.Status()
    abi.load().gwb_marginal_infeasibility(_ptr(p), p.shape[0], p.shape[1], _ptr(mu.weights()),
                                          mu.size(), _ptr(nu.weights()), nu.size(),
                                          C.byref(out), C.byref(st))
    abi.raise_for(st)
    return out.value


def split_gap(pi, w) -> float:
    """gw::split_gap (diagnostics.cpp:22-27)."""
    p, q = _f64(pi), _f64(w)
    if p.shape != q.shape:
        raise DimensionMismatchError("split_gap: shape mismatch")
    out = C.c_double(0.0)
    st = abi.Status()
    abi.load().gwb_split_gap(_ptr(p), _ptr(q), p.shape[0], p.shape[1], C.byref(out), C.byref(st))
    abi.raise_for(st)
    return out.value


def hard_assignment(pi) -> np.ndarray:
    """gw::hard_assignment (tasks.cpp:190-200)."""
    p = _f64(pi)
    out = np.empty(p.shape[0], dtype=np.int32)
    st = abi.Status()
    abi.load().gwb_hard_assignment(_ptr(p), p.shape[0], p.shape[1],
                                   out.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(st))
    abi.raise_for(st)
    return out


def coupling_entropy(pi) -> float:
    """gw::coupling_entropy (diagnostics.cpp:44-53): −Σ π log π, nats."""
    p = _f64(pi.entries() if isinstance(pi, Coupling) else pi)
    out, st = C.c_double(0), abi.Status()
    abi.load().gwb_coupling_entropy(_ptr(p), p.shape[0], p.shape[1], C.byref(out), C.byref(st))
    abi.raise_for(st)
    return out.value


def dykstra_project(pi, mu: ProbabilityVector, nu: ProbabilityVector, tol: float = 1e-8,
                    max_iters: int = 10000) -> np.ndarray:
    """gw::dykstra_project (projections.cpp:165-187): Euclidean projection onto
    Π(μ, ν); RuntimeError if the marginals do not reach `tol` in `max_iters`."""
    p = _f64(pi.entries() if isinstance(pi, Coupling) else pi)
    if p.shape != (mu.size(), nu.size()):
        raise DimensionMismatchError("dykstra_project: shape mismatch")
    out, st = np.empty_like(p, order="F"), abi.Status()
    abi.load().gwb_dykstra_project(_ptr(p), p.shape[0], p.shape[1], _ptr(mu.weights()),
                                   _ptr(nu.weights()), tol, max_iters, _ptr(out), C.byref(st))
    abi.raise_for(st)
    return out


def luo_tseng_residual(d_x: DistanceMatrix, d_y: DistanceMatrix, pi, mu: ProbabilityVector,
                       nu: ProbabilityVector, dykstra_tol: float = 1e-8) -> float:
    """gw::luo_tseng_residual (diagnostics.cpp:33-42):
    ‖π − dykstra_project(π + D_X π D_Y)‖_F."""
    p = _f64(pi.entries() if isinstance(pi, Coupling) else pi)
    if p.shape != (d_x.size(), d_y.size()):
        raise DimensionMismatchError("luo_tseng_residual: shape mismatch")
    out, st = C.c_double(0), abi.Status()
    abi.load().gwb_luo_tseng_residual(_ptr(d_x.entries()), d_x.size(), _ptr(d_y.entries()),
                                      d_y.size(), _ptr(p), _ptr(mu.weights()), _ptr(nu.weights()),
                                      dykstra_tol, C.byref(out), C.byref(st))
    abi.raise_for(st)
    return out.value


def format_coupling_csv(pi) -> bytes:
    """gw::write_coupling_csv (io.cpp:183-193) as bytes, formatted on the device."""
    p = _f64(pi.entries() if isinstance(pi, Coupling) else pi)
    n, m = p.shape
    ln, st = C.c_int64(0), abi.Status()
    lib = abi.load()
    lib.gwb_format_coupling_csv(_ptr(p), n, m, None, 0, C.byref(ln), C.byref(st))
    abi.raise_for(st)
    buf = C.create_string_buffer(max(1, ln.value))
    lib.gwb_format_coupling_csv(_ptr(p), n, m, buf, ln.value, C.byref(ln), C.byref(st))
    abi.raise_for(st)
    return buf.raw[: ln.value]


def write_coupling_csv_file(path: str, pi) -> None:
    """gw::write_coupling_csv_file (io.cpp:195-199)."""
    p = _f64(pi.entries() if isinstance(pi, Coupling) else pi)
    st = abi.Status()
    abi.load().gwb_write_coupling_csv_file(str(path).encode(), _ptr(p), p.shape[0], p.shape[1],
                                           C.byref(st))
    abi.raise_for(st)


def alignment_accuracy(pred, ground_truth) -> float:
    """gw::alignment_accuracy (tasks.cpp:202-214), percent."""
    a = np.ascontiguousarray(pred, dtype=np.int32)
    g = np.ascontiguousarray(ground_truth, dtype=np.int32)
    out, st = C.c_double(0), abi.Status()
    i32 = C.POINTER(C.c_int32)
    abi.load().gwb_alignment_accuracy(a.ctypes.data_as(i32), a.size, g.ctypes.data_as(i32), g.size,
                                      C.byref(out), C.byref(st))
    abi.raise_for(st)
    return out.value


def version() -> str:
    return abi.load().gwb_version().decode()
