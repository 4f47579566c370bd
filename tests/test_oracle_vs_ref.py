"""The C restatement (oracle/gw_oracle.c) against the reference's own
translation units (oracle/_ref) on seeded instances: every algorithm on the
path, traces, and error semantics.  Pins the oracle used by the GPU parity
tests.  Skipped where the reference is not buildable (the GPU box)."""
import numpy as np
import pytest

from paper_2205_08115_b200 import abi
from harness import instances as I

CASES = [
    ("bapg-er", lambda: I.config1(seed=1, n=96), dict(algorithm=abi.BAPG, rho=0.1, max_iters=40)),
    ("bapg-gmm", lambda: I.config2(seed=2, n=80, m=64), dict(algorithm=abi.BAPG, rho=0.05, max_iters=30)),
    ("bapg-sbm", lambda: I.config3(seed=3, n=120, k=6), dict(algorithm=abi.BAPG, rho=0.5, max_iters=30)),
    ("bapg-stop", lambda: I.config1(seed=4, n=64), dict(algorithm=abi.BAPG, rho=0.1, max_iters=500, rel_tol=1e-6)),
    ("ebpg", lambda: I.config1(seed=5, n=64), dict(algorithm=abi.EBPG, epsilon_reg=0.1, max_iters=15, inner_iters=10)),
    ("ebpg-log", lambda: I.config1(seed=6, n=64), dict(algorithm=abi.EBPG, epsilon_reg=0.01, log_domain=1, max_iters=10, inner_iters=20)),
    ("bpg", lambda: I.config1(seed=7, n=64), dict(algorithm=abi.BPG, step=5.0, max_iters=12, inner_iters=10)),
    ("hbpg", lambda: I.config1(seed=8, n=64), dict(algorithm=abi.HBPG, epsilon_reg=0.1, step=5.0, inner_iters=10, switch_iters=6, max_iters=14)),
    ("bpg-perturb", lambda: I.config1(seed=9, n=48), dict(algorithm=abi.BPG, perturbation=0.01, max_iters=8, inner_iters=20)),
    # quadratic geometry (euclid_project, projections.cpp:36-77; solvers.cpp:179-182)
    ("bapg-quad-er", lambda: I.config1(seed=10, n=72), dict(algorithm=abi.BAPG, geometry=abi.QUADRATIC, rho=0.1, max_iters=30)),
    ("bapg-quad-gmm", lambda: I.config2(seed=11, n=60, m=44), dict(algorithm=abi.BAPG, geometry=abi.QUADRATIC, rho=2.0, max_iters=40)),
    ("bapg-quad-stop", lambda: I.config1(seed=12, n=50), dict(algorithm=abi.BAPG, geometry=abi.QUADRATIC, rho=1.0, max_iters=400, rel_tol=1e-8)),
]


@pytest.mark.parametrize("name,make,over", CASES, ids=[c[0] for c in CASES])
def test_port_matches_reference(port, ref, name, make, over):
    inst = make()
    kw = dict(rel_tol=1e-30, quiet=1)
    kw.update(over)
    cfg = abi.default_config(**kw)
    a = port.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu)
    b = ref.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu)
    assert a.code == b.code == 0, (a.message, b.message)
    assert a.iterations_used == b.iterations_used and a.converged == b.converged
    scale = np.abs(b.final).max()
    assert np.abs(a.final - b.final).max() <= 1e-12 * scale
    assert len(a.trace) == len(b.trace)
    for x, y in zip(a.trace, b.trace):
        assert x["iter"] == y["iter"] and x["phase"] == y["phase"]
        for k in ("objective", "marginal_infeasibility", "split_gap", "rel_change"):
            assert x[k] == pytest.approx(y[k], rel=1e-9, abs=1e-15), (k, x[k], y[k])


@pytest.mark.parametrize("over,solver", [
    (dict(rho=1e-7), "bapg"),
    (dict(algorithm=abi.BPG, step=1e7, inner_iters=5), "bpg"),
    (dict(algorithm=abi.EBPG, epsilon_reg=1e-5, inner_iters=5), "ebpg"),
])
def test_error_semantics_match(port, ref, over, solver):
    inst = I.config1(seed=2, n=48)
    cfg = abi.default_config(rel_tol=1e-30, max_iters=5, quiet=1, **over)
    a = port.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu)
    b = ref.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu)
    assert a.code == b.code and a.message == b.message, (a.message, b.message)
    assert a.code == abi.ERR_NUMERICAL
    assert a.status.solver.decode() == solver


def test_initial_coupling_and_positivity(port, ref):
    inst = I.config1(seed=3, n=40)
    rng = np.random.default_rng(0)
    init = rng.random((40, 40)) + 0.1
    init /= init.sum()
    cfg = abi.default_config(rel_tol=1e-30, max_iters=5)
    a = port.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu, initial=init)
    b = ref.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu, initial=init)
    assert np.abs(a.final - b.final).max() <= 1e-13
    init[3, 4] = 0.0
    a = port.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu, initial=init)
    b = ref.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu, initial=init)
    assert a.code == b.code == abi.ERR_CONFIG and a.message == b.message


# ---- Luo-Tseng residual / Dykstra (diagnostics.cpp:33-42, projections.cpp:165-187)

def _residual_instance(seed=3, n=40, m=30):
    rng = np.random.default_rng(seed)
    dx = I.adjacency(n, I.erdos_renyi(n, 0.2, seed))
    dy = I.adjacency(m, I.erdos_renyi(m, 0.2, seed + 1))
    mu = rng.uniform(0.5, 1.5, n)
    nu = rng.uniform(0.5, 1.5, m)
    mu, nu = mu / mu.sum(), nu / nu.sum()
    pi = np.asfortranarray(np.outer(mu, nu) * rng.uniform(0.5, 1.5, (n, m)))
    return dx, dy, mu, nu, pi


def test_dykstra_and_residual_match_reference(port, ref):
    dx, dy, mu, nu, pi = _residual_instance()
    a, b = port.dykstra_project(3.0 * pi, mu, nu), ref.dykstra_project(3.0 * pi, mu, nu)
    assert a[0] == b[0] == 0
    assert np.abs(a[1] - b[1]).max() <= 1e-15
    ra, rb = port.luo_tseng_residual(dx, dy, pi, mu, nu), ref.luo_tseng_residual(dx, dy, pi, mu, nu)
    assert ra[0] == rb[0] == 0 and ra[1] == pytest.approx(rb[1], rel=1e-12)
    # non-convergence: runtime_error with the reference's message
    a, b = port.dykstra_project(3.0 * pi, mu, nu, max_iters=2), ref.dykstra_project(3.0 * pi, mu, nu, max_iters=2)
    assert a[0] == b[0] == abi.ERR_RUNTIME and a[2] == b[2]
    assert a[2].startswith("dykstra_project did not converge in 2 sweeps; final constraint violation")


@pytest.mark.parametrize("over", [
    dict(algorithm=abi.BAPG, rho=0.5),
    dict(algorithm=abi.BAPG, geometry=abi.QUADRATIC, rho=1.0),
    dict(algorithm=abi.HBPG, epsilon_reg=0.1, step=5.0, inner_iters=10, switch_iters=3),
], ids=["bapg", "bapg-quad", "hbpg"])
def test_record_residual_matches_reference(port, ref, over):
    dx, dy, mu, nu, _ = _residual_instance(seed=5, n=36, m=28)
    cfg = abi.default_config(rel_tol=1e-30, max_iters=6, quiet=1, record_residual=1, **over)
    a = port.solve(cfg, dx, dy, mu, nu)
    b = ref.solve(cfg, dx, dy, mu, nu)
    assert a.code == b.code == 0, (a.message, b.message)
    assert len(a.trace) == len(b.trace) == 6
    for x, y in zip(a.trace, b.trace):
        assert y["residual"] is not None
        assert x["residual"] == pytest.approx(y["residual"], rel=1e-10)


# ---- write_coupling_csv (io.cpp:183-193)

def csv_cases():
    rng = np.random.default_rng(17)
    big = rng.standard_normal((9, 7)) * 10.0 ** rng.integers(-320, 300, (9, 7))
    big.flat[:12] = [0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 2.2250738585072014e-308,
                     1.7976931348623157e308, 0.0001, 0.00001, 1e16, 1e17]
    # exact ties at the 17th digit: odd k · 2^-2 with 16 integer digits
    k = rng.integers(4 * 10**15, 9 * 10**15, 20) | 1
    ties = (k.astype(np.float64) / 4.0).reshape(4, 5)
    unit = rng.random((6, 11))
    return [big, ties, unit, np.ones((1, 1)), np.zeros((3, 0)), np.full((2, 3), 0.1)]


def test_coupling_csv_matches_reference(port, ref):
    for a in csv_cases():
        a = np.asfortranarray(a)
        assert port.format_coupling_csv(a) == ref.format_coupling_csv(a)
