"""Luo-Tseng residual (diagnostics.cpp:33-42) and Dykstra projection
(projections.cpp:165-187) on the device (csrc/residual.cu) against the CPU
oracle, whose restatement is pinned to the reference in
tests/test_oracle_vs_ref.py.  The residual takes one fp32-accumulated
(3xTF32) chain for D_X π D_Y and an fp64 Dykstra, so it is held to 1e-4
relative; the Dykstra projection alone is fp64 end to end (1e-12)."""
import numpy as np
import pytest

import paper_2205_08115_b200 as gw
from paper_2205_08115_b200 import abi
from harness import instances as I

pytestmark = pytest.mark.gpu


def _inst(seed, n, m, p=0.1):
    rng = np.random.default_rng(seed)
    dx = I.adjacency(n, I.erdos_renyi(n, p, seed))
    dy = I.adjacency(m, I.erdos_renyi(m, p, seed + 1))
    mu = rng.uniform(0.5, 1.5, n)
    nu = rng.uniform(0.5, 1.5, m)
    mu, nu = mu / mu.sum(), nu / nu.sum()
    pi = np.asfortranarray(np.outer(mu, nu) * rng.uniform(0.2, 1.8, (n, m)))
    return dx, dy, mu, nu, pi


@pytest.mark.parametrize("n,m", [(1, 1), (37, 29), (130, 97), (300, 300), (64, 1500),
                                 (1100, 40), (20, 5000), (24, 26000), (9, 60000), (13000, 6)])
def test_dykstra_project_matches_oracle(gpu, port, n, m):
    # Line blocks staged in shared memory across clusters of C CTAs (64 KB
    # per CTA): rows of length 1500 / 5000 / 26000 take C = 2 / 8 / 16;
    # 60000 exceeds a 16-CTA stage (global re-reads); columns of 13000
    # take C = 2.
    _, _, mu, nu, pi = _inst(n + m, n, m)
    x = gw.dykstra_project(2.5 * pi, gw.ProbabilityVector(mu), gw.ProbabilityVector(nu))
    rc, y, msg = port.dykstra_project(2.5 * pi, mu, nu)
    assert rc == 0, msg
    assert np.abs(x - y).max() <= 1e-12 * np.abs(y).max()
    assert np.abs(x.sum(axis=1) - mu).max() <= 1e-8
    assert np.abs(x.sum(axis=0) - nu).max() <= 1e-8


def test_dykstra_nonconvergence_message(gpu, port):
    _, _, mu, nu, pi = _inst(4, 50, 40)
    with pytest.raises(RuntimeError) as e:
        gw.dykstra_project(3.0 * pi, gw.ProbabilityVector(mu), gw.ProbabilityVector(nu),
                           max_iters=2)
    rc, _, msg = port.dykstra_project(3.0 * pi, mu, nu, max_iters=2)
    assert rc == abi.ERR_RUNTIME
    assert str(e.value) == msg


@pytest.mark.parametrize("n,m", [(40, 30), (257, 190), (500, 500)])
def test_luo_tseng_residual_matches_oracle(gpu, port, n, m):
    dx, dy, mu, nu, pi = _inst(7 + n, n, m)
    r = gw.luo_tseng_residual(gw.DistanceMatrix.trusted(dx), gw.DistanceMatrix.trusted(dy), pi,
                              gw.ProbabilityVector(mu), gw.ProbabilityVector(nu))
    rc, ro, msg = port.luo_tseng_residual(dx, dy, pi, mu, nu)
    assert rc == 0, msg
    assert abs(r - ro) <= 1e-4 * ro


def test_residual_non_binary_distances(gpu, port):
    g = I.config2(seed=3, n=150, m=120)  # Euclidean D: the 3xTF32 chain splits both operands
    rng = np.random.default_rng(1)
    pi = np.asfortranarray(np.outer(g.mu, g.nu) * rng.uniform(0.5, 1.5, (150, 120)))
    r = gw.luo_tseng_residual(gw.DistanceMatrix.trusted(g.dx), gw.DistanceMatrix.trusted(g.dy), pi,
                              gw.ProbabilityVector(g.mu), gw.ProbabilityVector(g.nu))
    rc, ro, msg = port.luo_tseng_residual(g.dx, g.dy, pi, g.mu, g.nu)
    assert rc == 0, msg
    assert abs(r - ro) <= 1e-4 * ro


def _check_trace(rep, o, tol=1e-4):
    assert len(rep.trace) == len(o.trace)
    for r, q in zip(rep.trace, o.trace):
        assert q["residual"] is not None and r.residual is not None
        assert abs(r.residual - q["residual"]) <= tol * q["residual"], (r.iter, r.residual, q["residual"])


@pytest.mark.parametrize("geometry,precision", [("entropy", "auto"), ("entropy", "sparse"),
                                                ("quadratic", "auto")])
def test_bapg_record_residual(gpu, port, geometry, precision):
    dx, dy, mu, nu, _ = _inst(21, 90, 70, p=0.15)
    cfg = gw.SolverConfig(geometry=geometry, rho=0.5, max_iters=8, rel_tol=1e-30, quiet=True,
                          record_residual=True, precision=precision)
    rep = gw.solve(gw.DistanceMatrix.trusted(dx), gw.DistanceMatrix.trusted(dy),
                   gw.ProbabilityVector(mu), gw.ProbabilityVector(nu), cfg)
    o = port.solve(cfg.to_abi(), dx, dy, mu, nu)
    assert o.code == 0, o.message
    _check_trace(rep, o)


def test_hbpg_record_residual(gpu, port):
    dx, dy, mu, nu, _ = _inst(22, 80, 64, p=0.15)
    cfg = gw.SolverConfig(algorithm="hbpg", epsilon_reg=0.1, step=5.0, inner_iters=10,
                          switch_iters=3, max_iters=6, rel_tol=1e-30, quiet=True,
                          record_residual=True)
    rep = gw.solve(gw.DistanceMatrix.trusted(dx), gw.DistanceMatrix.trusted(dy),
                   gw.ProbabilityVector(mu), gw.ProbabilityVector(nu), cfg)
    o = port.solve(cfg.to_abi(), dx, dy, mu, nu)
    assert o.code == 0, o.message
    _check_trace(rep, o)


def test_batched_record_residual(gpu, port):
    probs = [_inst(30 + k, 48, 48, p=0.2)[:4] for k in range(2)]
    cfg = gw.SolverConfig(rho=0.5, max_iters=5, rel_tol=1e-30, quiet=True, record_residual=True)
    reps = gw.bapg_solve_batched([gw.DistanceMatrix.trusted(p[0]) for p in probs],
                                 [gw.DistanceMatrix.trusted(p[1]) for p in probs],
                                 [gw.ProbabilityVector(p[2]) for p in probs],
                                 [gw.ProbabilityVector(p[3]) for p in probs], cfg)
    for rep, p in zip(reps, probs):
        o = port.solve(cfg.to_abi(), *p)
        _check_trace(rep, o)


def test_record_residual_off_leaves_it_empty(gpu):
    dx, dy, mu, nu, _ = _inst(23, 60, 50)
    cfg = gw.SolverConfig(rho=0.5, max_iters=3, rel_tol=1e-30, quiet=True)
    rep = gw.solve(gw.DistanceMatrix.trusted(dx), gw.DistanceMatrix.trusted(dy),
                   gw.ProbabilityVector(mu), gw.ProbabilityVector(nu), cfg)
    assert all(r.residual is None for r in rep.trace)
