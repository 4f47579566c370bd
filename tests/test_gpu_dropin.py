"""The compiled drop-in (dropin/gw_b200.cpp, built against the reference's
own headers and types.cpp, linked to libgwb.so) called with the reference's
C++ types: gw::bapg_solve / hbpg_solve / solve, gw::gw_objective,
gw::product_coupling, gw::lipschitz_bound (solvers.hpp:12-70,
types.hpp:177-178), the reference exception classes and validation order
(solvers.cpp:141-151), the observer and the initial coupling."""
import numpy as np
import pytest

from harness import cases as HC
from harness import instances as I
from paper_2205_08115_b200 import abi
from tests import dropin_lib as DL

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dl(gpu):
    return DL.load()


def cfg(**kw):
    kw.setdefault("quiet", 1)
    return abi.default_config(**kw)


def test_c1_bapg_solve_matches_port(dl, port):
    """The c1 config (ER n=1000, 2000 iterations) through gw::bapg_solve,
    against the reference fingerprint: objective and coupling bounds."""
    import os
    from tests.parity import QUANT, dequantise
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "fp_c1.npz"))
    inst, _ = HC.c1()
    c = cfg(**inst.solver)
    r = DL.solve(dl, "bapg", c, inst.dx, inst.dy, inst.mu, inst.nu)
    assert r["error"] is None, r["error"]
    assert r["iterations"] == int(z["iterations"]) == 2000
    obj, obj_ref = r["trace"][-1, 1], z["trace"][-1, 1]
    assert abs(obj - obj_ref) <= 1e-5 * abs(obj_ref)
    scale = float(z["scale"])
    assert np.abs(r["final"] - dequantise(z["q"], scale)).max() / scale + QUANT <= 1e-4
    # pi_half / w_half (solvers.cpp:214): rows of π sum to μ, columns of w to ν.
    np.testing.assert_allclose(r["pi"].sum(axis=1), inst.mu, rtol=1e-9)
    np.testing.assert_allclose(r["w"].sum(axis=0), inst.nu, rtol=1e-9)
    np.testing.assert_allclose(0.5 * (r["pi"] + r["w"]), r["final"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("entry,algorithm", [("solve", "hbpg"), ("hbpg", "hbpg"), ("solve", "ebpg"),
                                             ("bpg", "bpg")])
def test_bregman_entries_match_port(dl, port, entry, algorithm):
    inst = I.config1(seed=21, n=80)
    c = cfg(algorithm=algorithm, epsilon_reg=0.1, step=5.0, inner_iters=10, switch_iters=4,
            max_iters=8, rel_tol=1e-30)
    r = DL.solve(dl, entry, c, inst.dx, inst.dy, inst.mu, inst.nu)
    assert r["error"] is None, r["error"]
    o = port.solve(c, inst.dx, inst.dy, inst.mu, inst.nu)
    assert o.code == 0
    assert r["iterations"] == o.iterations_used
    assert np.abs(r["final"] - o.final).max() <= 1e-4 * np.abs(o.final).max()
    np.testing.assert_allclose(r["trace"][:, 1], [t["objective"] for t in o.trace], rtol=1e-5)
    np.testing.assert_array_equal(r["trace"][:, 5], [t["phase"] for t in o.trace])


def test_leaves_through_dropin(dl, port):
    d = np.array([[0.0, 1.0], [1.0, 0.0]])
    err, v = DL.gw_objective(dl, d, d, 0.5 * np.eye(2))
    assert err is None and abs(v + 0.5) <= 1e-12
    err, pc = DL.product_coupling(dl, [0.3, 0.7], [0.5, 0.5])
    assert err is None
    np.testing.assert_array_equal(pc, [[0.15, 0.15], [0.35, 0.35]])
    dx = I.adjacency(120, I.erdos_renyi(120, 0.08, 3))
    dy = I.adjacency(90, I.erdos_renyi(90, 0.08, 4))
    err, lip = DL.lipschitz_bound(dl, dx, dy)
    assert err is None and abs(lip - port.lipschitz_bound(dx, dy)) <= 1e-10 * lip
    rng = np.random.default_rng(5)
    pi = rng.uniform(0.5, 1.5, (120, 90))
    pi /= pi.sum()
    err, v = DL.gw_objective(dl, dx, dy, pi)
    rc, want, _ = port.gw_objective(dx, dy, pi)
    assert err is None and abs(v - want) <= 1e-5 * abs(want)  # 3xTF32 leaf, north-star bound


def test_validation_order_double_fault(dl, port):
    """A bad config AND mismatched sizes: ConfigError first (require_algorithm
    -> validate -> validate_inputs, solvers.cpp:141-143)."""
    inst = I.config1(seed=2, n=30)
    bad = cfg(rho=-1.0, max_iters=5)
    r = DL.solve(dl, "bapg", bad, inst.dx, inst.dy, inst.mu[:-1] / inst.mu[:-1].sum(), inst.nu)
    assert r["error"] == ("ConfigError", "rho must be positive")
    wrong = cfg(algorithm=abi.HBPG, rho=-1.0, max_iters=5)
    r = DL.solve(dl, "bapg", wrong, inst.dx, inst.dy, inst.mu, inst.nu)
    assert r["error"] == ("ConfigError", "bapg_solve called with algorithm 'hbpg'")
    r = DL.solve(dl, "bapg", cfg(max_iters=5), inst.dx, inst.dy,
                 inst.mu[:-1] / inst.mu[:-1].sum(), inst.nu)
    o = port.solve(cfg(max_iters=5), inst.dx, inst.dy, inst.mu, inst.nu)  # sanity: valid case ok
    assert o.code == 0
    assert r["error"] == ("DimensionMismatchError", "D_X is 30x30 but mu has length 29")
    r = DL.solve(dl, "bapg", cfg(max_iters=5), inst.dx, inst.dy, inst.mu, inst.nu,
                 initial=np.ones((30, 29)) / 870)
    assert r["error"] == ("DimensionMismatchError", "initial coupling shape mismatch")


def test_numerical_error_class_and_fields(dl, port):
    inst = I.config1(seed=2, n=64)
    c = cfg(rho=1e-6, max_iters=10)
    r = DL.solve(dl, "bapg", c, inst.dx, inst.dy, inst.mu, inst.nu)
    o = port.solve(c, inst.dx, inst.dy, inst.mu, inst.nu)
    assert o.code == abi.ERR_NUMERICAL
    assert r["error"] == ("NumericalInstabilityError", o.message)
    assert r["outcome"].solver.decode() == "bapg" and r["outcome"].iteration == o.status.iteration


def test_fw_stays_with_the_reference(dl):
    inst = I.config1(seed=2, n=16)
    r = DL.solve(dl, "solve", cfg(algorithm=abi.FW, max_iters=3), inst.dx, inst.dy, inst.mu,
                 inst.nu)
    assert r["error"][0] == "runtime_error" and "fw_solve" in r["error"][1]


@pytest.mark.parametrize("algorithm", [abi.BAPG, abi.HBPG])
def test_observer_and_initial_through_dropin(dl, port, algorithm):
    inst = I.config1(seed=8, n=72)
    init = I.jittered_product(inst.mu, inst.nu, 0.01, 5)
    c = cfg(algorithm=algorithm, epsilon_reg=0.1, step=5.0, inner_iters=10, switch_iters=3,
            max_iters=7, rel_tol=1e-30)
    r = DL.solve(dl, "solve", c, inst.dx, inst.dy, inst.mu, inst.nu, initial=init, observer=True)
    assert r["error"] is None, r["error"]
    # observer after every outer iteration; hBPG phase 2 numbered after phase 1
    assert list(r["observer_iters"]) == list(range(1, 8))
    mass = r["observer_mass"]
    want = 1.0 + (1e3 if algorithm == abi.BAPG else 0.0)  # Σπ (+ 1e3·Σw for BAPG)
    np.testing.assert_allclose(mass, want, rtol=1e-6)
    o = port.solve(c, inst.dx, inst.dy, inst.mu, inst.nu, initial=init)
    assert o.code == 0
    assert np.abs(r["final"] - o.final).max() <= 1e-4 * np.abs(o.final).max()
