"""ctypes access to the compiled drop-in (dropin/_build/libgw_dropin.so:
dropin/gw_b200.cpp + the reference's types.cpp, linked to libgwb.so).
Test infrastructure: calls the reference-signature gw:: entry points through
dropin/dropin_capi.cpp and returns what a C++ caller would observe."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "dropin", "_build", "libgw_dropin.so")
SYMBOLS = ["gwdi_solve", "gwdi_gw_objective", "gwdi_product_coupling", "gwdi_lipschitz_bound"]
ENTRY = {"solve": 0, "bapg": 1, "bpg": 2, "ebpg": 3, "hbpg": 4}


class Outcome(C.Structure):
    _fields_ = [("kind", C.c_char * 48), ("message", C.c_char * 512), ("solver", C.c_char * 16),
                ("iteration", C.c_int32), ("axis", C.c_int32), ("index", C.c_int64)]

    def error(self):
        k = self.kind.decode()
        return None if not k else (k, self.message.decode())


_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int32)


def load():
    if not os.path.exists(LIB):
        raise FileNotFoundError(f"{LIB} not built (dropin/Makefile, run by build())")
    lib = C.CDLL(LIB)
    lib.gwdi_solve.argtypes = [C.c_int32, _D, _D, C.c_int64, _D, C.c_int64, _D, C.c_int64, _D,
                               C.c_int64, _D, C.c_int64, C.c_int64, C.c_int32, _I, _D, C.c_int32,
                               _I, _D, _D, _D, _D, C.c_int32, _I, _I, _I, C.POINTER(Outcome)]
    lib.gwdi_gw_objective.argtypes = [_D, C.c_int64, _D, C.c_int64, _D, C.c_int64, C.c_int64, _D,
                                      C.POINTER(Outcome)]
    lib.gwdi_product_coupling.argtypes = [_D, C.c_int64, _D, C.c_int64, _D, C.POINTER(Outcome)]
    lib.gwdi_lipschitz_bound.argtypes = [_D, C.c_int64, _D, C.c_int64, _D, C.POINTER(Outcome)]
    return lib


def _f(a):
    return np.require(np.asarray(a, dtype=np.float64), requirements=["F_CONTIGUOUS", "ALIGNED"])


def _p(a):
    return None if a is None else a.ctypes.data_as(_D)


def config_vector(cfg) -> np.ndarray:
    """SolverConfig fields in types.hpp order from an abi.Config."""
    f = ["algorithm", "geometry", "rho", "step", "epsilon_reg", "inner_iters", "inner_tol",
         "rel_tol", "max_iters", "perturbation", "switch_iters", "seed", "log_domain",
         "record_residual"]
    return np.array([float(getattr(cfg, k)) for k in f])


def solve(lib, entry, cfg, dx, dy, mu, nu, initial=None, observer=False):
    dx, dy = _f(dx), _f(dy)
    mu, nu = np.ascontiguousarray(mu, float), np.ascontiguousarray(nu, float)
    n, m = dx.shape[0], dy.shape[0]
    init = None if initial is None else _f(initial)
    cap = max(1, int(cfg.max_iters))
    final = np.zeros((n, m), order="F")
    pi = np.zeros((n, m), order="F")
    w = np.zeros((n, m), order="F")
    trace = np.zeros((cap, 7))
    oi = np.zeros(cap + 8, dtype=np.int32)
    om = np.zeros(cap + 8)
    oc, nr, cv, used = C.c_int32(0), C.c_int32(0), C.c_int32(0), C.c_int32(0)
    out = Outcome()
    cv_ = config_vector(cfg)
    lib.gwdi_solve(ENTRY[entry], _p(cv_), _p(dx), n, _p(dy), m, _p(mu), mu.size, _p(nu), nu.size,
                   _p(init), 0 if init is None else init.shape[0],
                   0 if init is None else init.shape[1], int(observer), oi.ctypes.data_as(_I),
                   _p(om), oi.size, C.byref(oc), _p(final), _p(pi), _p(w), _p(trace), cap,
                   C.byref(nr), C.byref(cv), C.byref(used), C.byref(out))
    return dict(error=out.error(), outcome=out, final=final, pi=pi, w=w,
                trace=trace[: nr.value], converged=bool(cv.value), iterations=used.value,
                observer_iters=oi[: min(oc.value, oi.size)].copy(),
                observer_mass=om[: min(oc.value, om.size)].copy(), observer_calls=oc.value)


def gw_objective(lib, dx, dy, pi):
    dx, dy, pi = _f(dx), _f(dy), _f(pi)
    v, out = C.c_double(0), Outcome()
    lib.gwdi_gw_objective(_p(dx), dx.shape[0], _p(dy), dy.shape[0], _p(pi), pi.shape[0],
                          pi.shape[1], C.byref(v), C.byref(out))
    return out.error(), v.value


def product_coupling(lib, mu, nu):
    mu, nu = np.ascontiguousarray(mu, float), np.ascontiguousarray(nu, float)
    res, out = np.zeros((mu.size, nu.size), order="F"), Outcome()
    lib.gwdi_product_coupling(_p(mu), mu.size, _p(nu), nu.size, _p(res), C.byref(out))
    return out.error(), res


def lipschitz_bound(lib, dx, dy):
    dx, dy = _f(dx), _f(dy)
    v, out = C.c_double(0), Outcome()
    lib.gwdi_lipschitz_bound(_p(dx), dx.shape[0], _p(dy), dy.shape[0], C.byref(v), C.byref(out))
    return out.error(), v.value
