"""write_coupling_csv (io.cpp:183-193) formatted on the device (csrc/csv.cu)
against the oracle, whose "%.17g" restatement is pinned byte-for-byte to the
reference build in tests/test_oracle_vs_ref.py.  Bit-exact: the device does
the exact decimal conversion itself."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2205_08115_b200 as gw
from paper_2205_08115_b200 import abi
from harness import instances as I

from .test_oracle_vs_ref import csv_cases

pytestmark = pytest.mark.gpu


def test_csv_special_values_and_ties(gpu, port):
    for a in csv_cases():
        a = np.asfortranarray(a)
        assert gw.format_coupling_csv(a) == port.format_coupling_csv(a)


@pytest.mark.parametrize("exp_lo,exp_hi", [(-330, -290), (-20, 20), (280, 308), (-12, 0)])
def test_csv_random_bits(gpu, port, exp_lo, exp_hi):
    rng = np.random.default_rng(exp_lo + 1000)
    mant = rng.random((64, 33)) + 0.5
    a = np.asfortranarray(mant * 10.0 ** rng.integers(exp_lo, exp_hi, mant.shape)
                          * rng.choice([-1.0, 1.0], mant.shape))
    assert gw.format_coupling_csv(a) == port.format_coupling_csv(a)


def test_csv_raw_bit_patterns(gpu, port):
    # uniformly random 64-bit patterns: every exponent, subnormals, NaN payloads
    rng = np.random.default_rng(5)
    a = np.asfortranarray(rng.integers(0, 2**63, (128, 64), dtype=np.int64).view(np.float64))
    assert gw.format_coupling_csv(a) == port.format_coupling_csv(a)


def test_csv_of_a_solve_and_file(gpu, port, tmp_path):
    inst = I.config1(seed=3, n=257)
    rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                   gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu),
                   gw.SolverConfig(rho=0.1, max_iters=20, rel_tol=1e-30, quiet=True))
    plan = rep.final_coupling.entries()
    text = gw.format_coupling_csv(plan)
    assert text == port.format_coupling_csv(plan)
    path = tmp_path / "plan.csv"
    gw.write_coupling_csv_file(str(path), plan)
    assert path.read_bytes() == text
    with pytest.raises(RuntimeError, match="cannot write '/nonexistent-dir/x.csv'"):
        gw.write_coupling_csv_file("/nonexistent-dir/x.csv", plan)


def test_csv_capacity_error(gpu, port):
    a = np.asfortranarray(np.full((4, 4), 0.125))
    ln, st = C.c_int64(0), abi.Status()
    buf = C.create_string_buffer(8)
    abi.load().gwb_format_coupling_csv(a.ctypes.data_as(C.POINTER(C.c_double)), 4, 4, buf, 8,
                                       C.byref(ln), C.byref(st))
    assert st.code == abi.ERR_CAPACITY and ln.value == len(port.format_coupling_csv(a))


def test_session_csv_round_trips(gpu, port, tmp_path):
    import torch
    inst = I.config1(seed=4, n=200)
    n = inst.n
    ld = (n + 31) // 32 * 32
    t = lambda x: torch.nn.functional.pad(torch.tensor(np.ascontiguousarray(x), dtype=torch.float32),
                                          (0, ld - x.shape[1])).cuda()
    dx, dy = t(inst.dx), t(inst.dy)
    mu = torch.tensor(inst.mu, dtype=torch.float32).cuda()
    lib = abi.load()
    cfg = abi.default_config(rho=0.1, max_iters=30, rel_tol=1e-30)
    st, s = abi.Status(), C.c_void_p()
    lib.gwb_session_create(C.byref(cfg), n, n, 0, C.byref(s), C.byref(st))
    abi.raise_for(st)
    path = tmp_path / "session.csv"
    try:
        lib.gwb_session_load_device(s, dx.data_ptr(), ld, dy.data_ptr(), ld, mu.data_ptr(),
                                    mu.data_ptr(), None, C.byref(st))
        lib.gwb_session_reset(s, None, C.byref(st))
        lib.gwb_session_iterate(s, 30, None, None, C.byref(st))
        abi.raise_for(st)
        lib.gwb_session_write_coupling_csv(s, str(path).encode(), C.byref(st))
        abi.raise_for(st)
    finally:
        lib.gwb_session_destroy(s)
    raw = path.read_bytes()
    lines = raw.decode().splitlines()
    assert lines[0] == f"{n},{n}"
    plan = np.asfortranarray(np.array([[float(v) for v in ln.split(",")] for ln in lines[1:]]))
    assert port.format_coupling_csv(plan) == raw  # the parse round-trips byte for byte
    o = port.solve(abi.default_config(rho=0.1, max_iters=30, rel_tol=1e-30), inst.dx, inst.dy,
                   inst.mu, inst.nu)
    assert np.abs(plan - o.final).max() <= 1e-4 * np.abs(o.final).max()
