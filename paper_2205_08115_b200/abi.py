"""ctypes mirror of the C-ABI in ``include/gwb.h`` and the exception mapping.

The structs here are byte-compatible with the header; the exception classes
mirror the reference hierarchy (``/root/reference/proj/include/gw/types.hpp:27-59``)
so callers and tests catch the same types the reference throws.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgwb.so")

# enums (gwb.h)
BAPG, BPG, EBPG, HBPG, FW = 0, 1, 2, 3, 4
ENTROPY, QUADRATIC = 0, 1
ROWS, COLS = 0, 1
(PREC_AUTO, PREC_TF32, PREC_3XTF32, PREC_BF16X3, PREC_BF16X2, PREC_SPARSE, PREC_FP32, PREC_F16X2,
 PREC_F16X3) = range(9)

OK = 0
ERR_CONFIG, ERR_DIMENSION, ERR_NUMERICAL, ERR_ZERO_SUM = 1, 2, 3, 4
ERR_INVALID, ERR_DOMAIN, ERR_UNSUPPORTED, ERR_RUNTIME, ERR_CAPACITY = 5, 6, 7, 8, 9

ALGORITHMS = {"bapg": BAPG, "bpg": BPG, "ebpg": EBPG, "hbpg": HBPG, "fw": FW}


class Config(C.Structure):
    """gwb_config == gw::SolverConfig (types.hpp:132-147) + B200 extensions."""

    _fields_ = [
        ("algorithm", C.c_int32),
        ("geometry", C.c_int32),
        ("rho", C.c_double),
        ("step", C.c_double),
        ("epsilon_reg", C.c_double),
        ("inner_iters", C.c_int32),
        ("inner_tol", C.c_double),
        ("rel_tol", C.c_double),
        ("max_iters", C.c_int32),
        ("perturbation", C.c_double),
        ("switch_iters", C.c_int32),
        ("seed", C.c_int64),
        ("log_domain", C.c_int32),
        ("record_residual", C.c_int32),
        ("precision", C.c_int32),
        ("quiet", C.c_int32),
    ]


class Readout(C.Structure):
    """gwb_readout: run_cell's post-solve readout (experiment.cpp:169-195)."""

    _fields_ = [
        ("objective", C.c_double),
        ("marginal_infeasibility", C.c_double),
        ("entropy", C.c_double),
        ("split_gap", C.c_double),
        ("residual", C.c_double),
        ("accuracy", C.c_double),
        ("has_accuracy", C.c_int32),
    ]


def default_config(**kw) -> Config:
    """SolverConfig defaults (types.hpp:132-147; test_core.cpp:145-159)."""
    c = Config(
        algorithm=BAPG, geometry=ENTROPY, rho=0.1, step=5.0, epsilon_reg=0.1,
        inner_iters=1000, inner_tol=1e-9, rel_tol=1e-6, max_iters=2000,
        perturbation=0.0, switch_iters=200, seed=0, log_domain=0,
        record_residual=0, precision=PREC_AUTO, quiet=0,
    )
    for k, v in kw.items():
        if k == "algorithm" and isinstance(v, str):
            v = ALGORITHMS[v]
        setattr(c, k, v)
    return c


class Record(C.Structure):
    """gwb_record == gw::IterationRecord (types.hpp:152-161)."""

    _fields_ = [
        ("iter", C.c_int32),
        ("objective", C.c_double),
        ("marginal_infeasibility", C.c_double),
        ("split_gap", C.c_double),
        ("residual", C.c_double),
        ("has_residual", C.c_int32),
        ("rel_change", C.c_double),
        ("elapsed_seconds", C.c_double),
        ("phase", C.c_int32),
    ]


class Status(C.Structure):
    _fields_ = [
        ("code", C.c_int32),
        ("iteration", C.c_int32),
        ("axis", C.c_int32),
        ("index", C.c_int64),
        ("solver", C.c_char * 16),
        ("message", C.c_char * 512),
    ]


OBSERVER = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int32, C.POINTER(C.c_double),
                       C.POINTER(C.c_double), C.c_int64, C.c_int64)


# --- exception hierarchy (types.hpp:27-59) ---------------------------------
class ConfigError(ValueError):
    """gw::ConfigError (std::invalid_argument)."""


class DimensionMismatchError(ValueError):
    """gw::DimensionMismatchError (std::invalid_argument)."""


class ZeroSumLineError(RuntimeError):
    """gw::ZeroSumLineError (std::runtime_error); carries axis and index."""

    def __init__(self, msg, axis=ROWS, index=0):
        super().__init__(msg)
        self.axis = axis
        self.index = index


class NumericalInstabilityError(RuntimeError):
    """gw::NumericalInstabilityError (std::runtime_error)."""

    def __init__(self, msg, solver="", iteration=0):
        super().__init__(msg)
        self.solver = solver
        self.iteration = iteration


class UnsupportedError(NotImplementedError):
    """Outside the B200 path (FW, quadratic geometry, Luo-Tseng residual)."""


class DomainError(ValueError):
    """std::domain_error."""


def raise_for(st: Status):
    """Rethrow a gwb_status as the reference exception class."""
    code = st.code
    if code == OK:
        return
    msg = st.message.decode(errors="replace")
    if code == ERR_CONFIG:
        raise ConfigError(msg)
    if code == ERR_DIMENSION:
        raise DimensionMismatchError(msg)
    if code == ERR_NUMERICAL:
        raise NumericalInstabilityError(msg, st.solver.decode(), st.iteration)
    if code == ERR_ZERO_SUM:
        raise ZeroSumLineError(msg, st.axis, st.index)
    if code == ERR_INVALID:
        raise ValueError(msg)
    if code == ERR_DOMAIN:
        raise DomainError(msg)
    if code == ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise RuntimeError(msg or f"gwb error code {code}")


# --- signatures ------------------------------------------------------------
_D = C.POINTER(C.c_double)
_F = C.POINTER(C.c_float)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)
_ST = C.POINTER(Status)

SOLVE_ARGS = [C.POINTER(Config), _D, C.c_int64, _D, C.c_int64, _D, _D, _D,
              OBSERVER, C.c_void_p, _D, _D, _D, C.POINTER(Record), C.c_int32,
              _I32, _I32, _I32, _ST]

SIGNATURES = {
    "gwb_config_default": (None, [C.POINTER(Config)]),
    "gwb_validate_config": (C.c_int32, [C.POINTER(Config), _ST]),
    "gwb_solve": (C.c_int32, SOLVE_ARGS),
    "gwb_bapg_solve": (C.c_int32, SOLVE_ARGS),
    "gwb_bpg_solve": (C.c_int32, SOLVE_ARGS),
    "gwb_ebpg_solve": (C.c_int32, SOLVE_ARGS),
    "gwb_hbpg_solve": (C.c_int32, SOLVE_ARGS),
    "gwb_gw_objective": (C.c_int32, [_D, C.c_int64, _D, C.c_int64, _D, C.c_int64,
                                     C.c_int64, _D, _ST]),
    "gwb_product_coupling": (C.c_int32, [_D, C.c_int64, _D, C.c_int64, _D, _ST]),
    "gwb_lipschitz_bound": (C.c_int32, [_D, C.c_int64, _D, C.c_int64, _D, _ST]),
    "gwb_kl_scale": (C.c_int32, [_D, C.c_int64, C.c_int64, _D, C.c_int64,
                                 C.c_int32, _D, _ST]),
    "gwb_sinkhorn_project": (C.c_int32, [_D, C.c_int64, C.c_int64, _D, _D,
                                         C.c_double, C.c_int32, C.c_int32, _D,
                                         _I32, _D, _I32, _ST]),
    "gwb_marginal_infeasibility": (C.c_int32, [_D, C.c_int64, C.c_int64, _D,
                                               C.c_int64, _D, C.c_int64, _D, _ST]),
    "gwb_split_gap": (C.c_int32, [_D, _D, C.c_int64, C.c_int64, _D, _ST]),
    "gwb_hard_assignment": (C.c_int32, [_D, C.c_int64, C.c_int64, _I32, _ST]),
    "gwb_coupling_entropy": (C.c_int32, [_D, C.c_int64, C.c_int64, _D, _ST]),
    "gwb_format_coupling_csv": (C.c_int32, [_D, C.c_int64, C.c_int64, C.c_char_p, C.c_int64,
                                            C.POINTER(C.c_int64), _ST]),
    "gwb_write_coupling_csv_file": (C.c_int32, [C.c_char_p, _D, C.c_int64, C.c_int64, _ST]),
    "gwb_session_write_coupling_csv": (C.c_int32, [C.c_void_p, C.c_char_p, _ST]),
    "gwb_dykstra_last_stats": (C.c_int32, [C.POINTER(C.c_int32), _D]),
    "gwb_dykstra_project": (C.c_int32, [_D, C.c_int64, C.c_int64, _D, _D, C.c_double, C.c_int32,
                                        _D, _ST]),
    "gwb_luo_tseng_residual": (C.c_int32, [_D, C.c_int64, _D, C.c_int64, _D, _D, _D, C.c_double,
                                           _D, _ST]),
    "gwb_session_readout": (C.c_int32, [C.c_void_p, _I32, C.c_int64, _I32, C.POINTER(Readout),
                                        _ST]),
    "gwb_alignment_accuracy": (C.c_int32, [_I32, C.c_int64, _I32, C.c_int64, _D, _ST]),
    "gwb_solve_graphs": (C.c_int32, [C.POINTER(Config), C.c_int64, C.POINTER(C.c_int32),
                                     C.c_int64, C.c_int64, C.POINTER(C.c_int32), C.c_int64,
                                     _D, _D, _D, OBSERVER, C.c_void_p, _D, _D, _D,
                                     C.POINTER(Record), C.c_int32, _I32, _I32, _I32, _ST]),
    "gwb_bapg_solve_batched": (C.c_int32, [C.POINTER(Config), C.c_int64, _D,
                                           C.c_int64, _D, C.c_int64, _D, _D, _D,
                                           _D, _D, C.POINTER(Record), C.c_int32,
                                           _I32, _I32, _I32, _ST]),
    "gwb_set_devices": (C.c_int32, [C.c_int32, _I32, _ST]),
    "gwb_session_create": (C.c_int32, [C.POINTER(Config), C.c_int64, C.c_int64,
                                       C.c_int32, C.POINTER(C.c_void_p), _ST]),
    "gwb_session_load_device": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int64,
                                            C.c_void_p, C.c_int64, C.c_void_p,
                                            C.c_void_p, C.c_void_p, _ST]),
    "gwb_session_reset": (C.c_int32, [C.c_void_p, C.c_void_p, _ST]),
    "gwb_session_iterate": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p,
                                        _I64, _ST]),
    "gwb_session_pi": (C.c_int32, [C.c_void_p, C.POINTER(C.c_void_p), _I64, _ST]),
    "gwb_session_kernel_ms": (C.c_int32, [C.c_void_p, C.c_int32, _D, _I64, _ST]),
    "gwb_session_destroy": (C.c_int32, [C.c_void_p]),
    "gwb_version": (C.c_char_p, []),
}

_LIB = None


def load(path: str | None = None) -> C.CDLL:
    """Load libgwb.so (built in-tree by __graft_entry__.build()).

    Fails loudly when the extension is missing: there is no CPU fallback.
    """
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (no CPU fallback exists for the GW solver path)")
    lib = C.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib
