"""ctypes access to the CPU checkers — TEST INFRASTRUCTURE ONLY.

``Oracle("port")`` wraps oracle/libgworacle.so (the C restatement);
``Oracle("reference")`` wraps oracle/_ref/libgwref.so (the reference's own
translation units compiled against eigen_lite).  Only tests/, smoke() and
bench.py's cpu_baseline leg may use this module.
"""
from __future__ import annotations

import ctypes as C
import glob
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from paper_2205_08115_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "libgworacle.so")
REF_LIB = os.path.join(HERE, "_ref", "libgwref.so")


def openblas_path() -> Optional[str]:
    import numpy
    libs = glob.glob(os.path.join(os.path.dirname(numpy.__file__) + ".libs", "libscipy_openblas64_*.so"))
    return libs[0] if libs else None


_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int32)
_ST = C.POINTER(abi.Status)
_SOLVE = [C.POINTER(abi.Config), _D, C.c_int64, _D, C.c_int64, _D, _D, _D, _D, _D, _D,
          C.POINTER(abi.Record), C.c_int32, _I, _I, _I, _ST]


def _p(a):
    return None if a is None else a.ctypes.data_as(_D)


def _f(a):
    return np.require(np.asarray(a, dtype=np.float64), requirements=["F_CONTIGUOUS", "ALIGNED"])


@dataclass
class OracleResult:
    code: int
    message: str
    final: Optional[np.ndarray] = None
    pi: Optional[np.ndarray] = None
    w: Optional[np.ndarray] = None
    trace: List[dict] = field(default_factory=list)
    converged: bool = False
    iterations_used: int = 0
    status: Optional[abi.Status] = None


class Oracle:
    def __init__(self, kind: str = "port", blas: bool = True):
        self.kind = kind
        blas_path = openblas_path() if blas else None
        if kind == "reference":
            if blas_path:
                os.environ.setdefault("GWREF_BLAS", blas_path)
            if not os.path.exists(REF_LIB):
                raise FileNotFoundError(f"{REF_LIB} not built (oracle/Makefile `ref` target)")
            self.lib = C.CDLL(REF_LIB)
            pre = "gwref_"
        else:
            self.lib = C.CDLL(PORT_LIB)
            pre = "gwo_"
            if blas_path:
                self._blas = C.CDLL(blas_path)
                self.lib.gwo_set_dgemm.argtypes = [C.c_void_p]
                self.lib.gwo_set_dgemm(C.cast(self._blas.scipy_cblas_dgemm64_, C.c_void_p))
        self.pre = pre
        L = self.lib
        getattr(L, pre + "solve").argtypes = _SOLVE
        getattr(L, pre + "solve").restype = C.c_int32
        getattr(L, pre + "gw_objective").argtypes = [_D, C.c_int64, _D, C.c_int64, _D, C.c_int64, C.c_int64, _D, _ST]
        getattr(L, pre + "product_coupling").argtypes = [_D, C.c_int64, _D, C.c_int64, _D, _ST]
        getattr(L, pre + "kl_scale").argtypes = [_D, C.c_int64, C.c_int64, _D, C.c_int64, C.c_int32, _D, _ST]
        getattr(L, pre + "sinkhorn_project").argtypes = [_D, C.c_int64, C.c_int64, _D, _D, C.c_double,
                                                C.c_int32, C.c_int32, _D, _I, _D, _I, _ST]
        getattr(L, pre + "dykstra_project").argtypes = [_D, C.c_int64, C.c_int64, _D, _D, C.c_double,
                                                        C.c_int32, _D, _I, _ST]
        getattr(L, pre + "luo_tseng_residual").argtypes = [_D, C.c_int64, _D, C.c_int64, _D, _D, _D,
                                                           C.c_double, _D, _ST]
        getattr(L, pre + "format_coupling_csv").argtypes = [_D, C.c_int64, C.c_int64, C.c_char_p,
                                                            C.c_int64, C.POINTER(C.c_int64), _ST]
        if kind == "reference":
            L.gwref_lipschitz_bound.argtypes = [_D, C.c_int64, _D, C.c_int64, _D, _ST]
            L.gwref_marginal_infeasibility.argtypes = [_D, C.c_int64, C.c_int64, _D, _D, _D, _ST]
            L.gwref_split_gap.argtypes = [_D, _D, C.c_int64, C.c_int64, _D, _ST]
            L.gwref_hard_assignment.argtypes = [_D, C.c_int64, C.c_int64, _I, _ST]
            L.gwref_coupling_entropy.argtypes = [_D, C.c_int64, C.c_int64, _D, _ST]
            L.gwref_alignment_accuracy.argtypes = [_I, C.c_int64, _I, C.c_int64, _D, _ST]
        else:
            L.gwo_lipschitz_bound.argtypes = [_D, C.c_int64, _D, C.c_int64]
            L.gwo_lipschitz_bound.restype = C.c_double
            L.gwo_marginal_infeasibility.argtypes = [_D, C.c_int64, C.c_int64, _D, _D]
            L.gwo_marginal_infeasibility.restype = C.c_double
            L.gwo_split_gap.argtypes = [_D, _D, C.c_int64, C.c_int64]
            L.gwo_split_gap.restype = C.c_double
            L.gwo_hard_assignment.argtypes = [_D, C.c_int64, C.c_int64, _I]
            L.gwo_coupling_entropy.argtypes = [_D, C.c_int64, C.c_int64]
            L.gwo_coupling_entropy.restype = C.c_double
            L.gwo_alignment_accuracy.argtypes = [_I, C.c_int64, _I, C.c_int64, _D, _ST]

    # -- solver -------------------------------------------------------------
    def solve(self, cfg: abi.Config, dx, dy, mu, nu, initial=None) -> OracleResult:
        dx, dy = _f(dx), _f(dy)
        mu, nu = np.ascontiguousarray(mu, dtype=np.float64), np.ascontiguousarray(nu, dtype=np.float64)
        n, m = dx.shape[0], dy.shape[0]
        init = None if initial is None else _f(initial)
        final = np.empty((n, m), order="F")
        pi = np.empty((n, m), order="F")
        w = np.empty((n, m), order="F")
        cap = max(1, cfg.max_iters)
        trace = (abi.Record * cap)()
        nr, cv, used = C.c_int32(0), C.c_int32(0), C.c_int32(0)
        st = abi.Status()
        rc = getattr(self.lib, self.pre + "solve")(C.byref(cfg), _p(dx), n, _p(dy), m, _p(mu), _p(nu),
                                          _p(init), _p(final), _p(pi), _p(w), trace, cap,
                                          C.byref(nr), C.byref(cv), C.byref(used), C.byref(st))
        res = OracleResult(rc, st.message.decode(errors="replace"), status=st)
        if rc == abi.OK:
            res.final, res.converged, res.iterations_used = final, bool(cv.value), used.value
            if cfg.algorithm == abi.BAPG:
                res.pi, res.w = pi, w
            res.trace = [dict(iter=r.iter, objective=r.objective,
                              marginal_infeasibility=r.marginal_infeasibility,
                              split_gap=r.split_gap, rel_change=r.rel_change,
                              elapsed_seconds=r.elapsed_seconds, phase=r.phase,
                              residual=r.residual if r.has_residual else None)
                         for r in trace[: nr.value]]
        return res

    # -- leaves -------------------------------------------------------------
    def gw_objective(self, dx, dy, pi):
        dx, dy, pi = _f(dx), _f(dy), _f(pi)
        out, st = C.c_double(0), abi.Status()
        rc = getattr(self.lib, self.pre + "gw_objective")(_p(dx), dx.shape[0], _p(dy), dy.shape[0], _p(pi),
                                                 pi.shape[0], pi.shape[1], C.byref(out), C.byref(st))
        return rc, out.value, st

    def product_coupling(self, mu, nu):
        mu, nu = np.ascontiguousarray(mu, float), np.ascontiguousarray(nu, float)
        out, st = np.empty((mu.size, nu.size), order="F"), abi.Status()
        rc = getattr(self.lib, self.pre + "product_coupling")(_p(mu), mu.size, _p(nu), nu.size, _p(out), C.byref(st))
        return rc, out, st

    def kl_scale(self, pi, target, axis):
        pi, t = _f(pi), np.ascontiguousarray(target, float)
        out, st = np.empty_like(pi, order="F"), abi.Status()
        rc = getattr(self.lib, self.pre + "kl_scale")(_p(pi), pi.shape[0], pi.shape[1], _p(t), t.size, axis,
                                             _p(out), C.byref(st))
        return rc, out, st

    def sinkhorn(self, kernel, mu, nu, tol, max_iters, log_domain=False):
        k = _f(kernel)
        mu, nu = np.ascontiguousarray(mu, float), np.ascontiguousarray(nu, float)
        out, st = np.empty_like(k, order="F"), abi.Status()
        it, err, cv = C.c_int32(0), C.c_double(0), C.c_int32(0)
        rc = getattr(self.lib, self.pre + "sinkhorn_project")(_p(k), k.shape[0], k.shape[1], _p(mu), _p(nu),
                                                     tol, max_iters, int(log_domain), _p(out),
                                                     C.byref(it), C.byref(err), C.byref(cv), C.byref(st))
        return rc, dict(coupling=out, iterations=it.value, marginal_error=err.value,
                        converged=bool(cv.value)), st

    def dykstra_project(self, pi, mu, nu, tol=1e-8, max_iters=10000):
        """Returns (code, projected coupling, message)."""
        pi = _f(pi)
        mu, nu = np.ascontiguousarray(mu, float), np.ascontiguousarray(nu, float)
        out, st, sw = np.empty_like(pi, order="F"), abi.Status(), C.c_int32(0)
        rc = getattr(self.lib, self.pre + "dykstra_project")(_p(pi), pi.shape[0], pi.shape[1], _p(mu),
                                                            _p(nu), tol, max_iters, _p(out),
                                                            C.byref(sw), C.byref(st))
        return rc, out, st.message.decode(errors="replace")

    def luo_tseng_residual(self, dx, dy, pi, mu, nu, tol=1e-8):
        """Returns (code, residual, message)."""
        dx, dy, pi = _f(dx), _f(dy), _f(pi)
        mu, nu = np.ascontiguousarray(mu, float), np.ascontiguousarray(nu, float)
        out, st = C.c_double(0), abi.Status()
        rc = getattr(self.lib, self.pre + "luo_tseng_residual")(_p(dx), dx.shape[0], _p(dy), dy.shape[0],
                                                               _p(pi), _p(mu), _p(nu), tol,
                                                               C.byref(out), C.byref(st))
        return rc, out.value, st.message.decode(errors="replace")

    def format_coupling_csv(self, pi) -> bytes:
        """write_coupling_csv (io.cpp:183-193) as bytes."""
        pi = _f(pi)
        n, m = pi.shape
        ln, st = C.c_int64(0), abi.Status()
        fn = getattr(self.lib, self.pre + "format_coupling_csv")
        fn(_p(pi), n, m, None, 0, C.byref(ln), C.byref(st))
        buf = C.create_string_buffer(max(1, ln.value))
        fn(_p(pi), n, m, buf, ln.value, C.byref(ln), C.byref(st))
        return buf.raw[: ln.value]

    def lipschitz_bound(self, dx, dy):
        dx, dy = _f(dx), _f(dy)
        if self.kind == "reference":
            out, st = C.c_double(0), abi.Status()
            self.lib.gwref_lipschitz_bound(_p(dx), dx.shape[0], _p(dy), dy.shape[0], C.byref(out), C.byref(st))
            return out.value
        return self.lib.gwo_lipschitz_bound(_p(dx), dx.shape[0], _p(dy), dy.shape[0])

    def marginal_infeasibility(self, pi, mu, nu):
        pi = _f(pi)
        mu, nu = np.ascontiguousarray(mu, float), np.ascontiguousarray(nu, float)
        if self.kind == "reference":
            out, st = C.c_double(0), abi.Status()
            self.lib.gwref_marginal_infeasibility(_p(pi), pi.shape[0], pi.shape[1], _p(mu), _p(nu),
                                                  C.byref(out), C.byref(st))
            return out.value
        return self.lib.gwo_marginal_infeasibility(_p(pi), pi.shape[0], pi.shape[1], _p(mu), _p(nu))

    def split_gap(self, pi, w):
        pi, w = _f(pi), _f(w)
        if self.kind == "reference":
            out, st = C.c_double(0), abi.Status()
            self.lib.gwref_split_gap(_p(pi), _p(w), pi.shape[0], pi.shape[1], C.byref(out), C.byref(st))
            return out.value
        return self.lib.gwo_split_gap(_p(pi), _p(w), pi.shape[0], pi.shape[1])

    def hard_assignment(self, pi):
        pi = _f(pi)
        out = np.empty(pi.shape[0], dtype=np.int32)
        if self.kind == "reference":
            st = abi.Status()
            self.lib.gwref_hard_assignment(_p(pi), pi.shape[0], pi.shape[1],
                                           out.ctypes.data_as(_I), C.byref(st))
        else:
            self.lib.gwo_hard_assignment(_p(pi), pi.shape[0], pi.shape[1], out.ctypes.data_as(_I))
        return out


    def coupling_entropy(self, pi):
        pi = _f(pi)
        if self.kind == "reference":
            out, st = C.c_double(0), abi.Status()
            self.lib.gwref_coupling_entropy(_p(pi), pi.shape[0], pi.shape[1], C.byref(out), C.byref(st))
            return out.value
        return self.lib.gwo_coupling_entropy(_p(pi), pi.shape[0], pi.shape[1])

    def alignment_accuracy(self, pred, gt):
        """Returns (code, accuracy %, message)."""
        pred = np.ascontiguousarray(pred, dtype=np.int32)
        gt = np.ascontiguousarray(gt, dtype=np.int32)
        out, st = C.c_double(0), abi.Status()
        rc = getattr(self.lib, self.pre + "alignment_accuracy")(
            pred.ctypes.data_as(_I), pred.size, gt.ctypes.data_as(_I), gt.size, C.byref(out),
            C.byref(st))
        return rc, out.value, st.message.decode(errors="replace")


def reference_generators():
    """The reference's own generators (tasks.cpp) for pinning instances.py."""
    lib = Oracle("reference", blas=False).lib
    I32, I64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64)
    lib.gwref_gen_barabasi_albert.argtypes = [C.c_int32, C.c_int32, C.c_uint64, I32, C.c_int64, I64, _ST]
    lib.gwref_gen_gaussian_partition.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double,
                                                 C.c_uint64, I32, C.c_int64, I64, I32, _ST]
    lib.gwref_permute_graph.argtypes = [C.c_int64, I32, C.c_int64, C.c_uint64, I32, I32, _ST]
    lib.gwref_adjacency_distance.argtypes = [C.c_int64, I32, C.c_int64, _D, _ST]
    return lib
