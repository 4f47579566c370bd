"""BAPG with the quadratic (Euclidean) geometry (csrc/quadratic.cu) against
the CPU oracle, whose restatement (sort-based simplex_project,
projections.cpp:36-77) is pinned to the reference in
tests/test_oracle_vs_ref.py.  Same bounds as the entropy path."""
import numpy as np
import pytest

import paper_2205_08115_b200 as gw
from harness import instances as I

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def run(port, dx, dy, mu, nu, initial=None, **solver):
    cfg = gw.SolverConfig(geometry="quadratic", quiet=True, **solver)
    opts = gw.SolveOptions(initial=initial) if initial is not None else None
    rep = gw.solve(gw.DistanceMatrix.trusted(dx), gw.DistanceMatrix.trusted(dy),
                   gw.ProbabilityVector(mu), gw.ProbabilityVector(nu), cfg, opts)
    o = port.solve(cfg.to_abi(), dx, dy, mu, nu, initial)
    assert o.code == 0, o.message
    assert rep.iterations_used == o.iterations_used
    assert rep.converged == o.converged
    assert rel(rep.final_coupling.entries(), o.final) < 1e-4
    assert rel(rep.pi_half.entries(), o.pi) < 1e-4
    assert rel(rep.w_half.entries(), o.w) < 1e-4
    obj, obj_ref = rep.trace[-1].objective, o.trace[-1]["objective"]
    assert abs(obj - obj_ref) <= 1e-5 * abs(obj_ref)
    for r, q in zip(rep.trace, o.trace):  # per-iteration records: as the entropy tests
        assert abs(r.objective - q["objective"]) <= 2e-4 * abs(q["objective"])
        assert abs(r.split_gap - q["split_gap"]) <= 1e-3 * q["split_gap"] + 1e-7
    return rep, o


@pytest.mark.parametrize("precision", ["auto", "sparse"])
def test_quadratic_er(gpu, port, precision):
    inst = I.config1(seed=10, n=300)
    run(port, inst.dx, inst.dy, inst.mu, inst.nu, rho=1.0, max_iters=40, rel_tol=1e-30,
        precision=precision)


def test_quadratic_weighted_gmm(gpu, port):
    g = I.config2(seed=11, n=200, m=150)
    run(port, g.dx, g.dy, g.mu, g.nu, rho=2.0, max_iters=40, rel_tol=1e-30)


def test_quadratic_ragged_nonuniform_and_initial(gpu, port):
    rng = np.random.default_rng(5)
    n, m = 130, 97
    dx = I.adjacency(n, I.erdos_renyi(n, 0.06, 31))
    dy = I.adjacency(m, I.erdos_renyi(m, 0.08, 32))
    mu = rng.uniform(0.5, 1.5, n)
    nu = rng.uniform(0.5, 1.5, m)
    mu, nu = mu / mu.sum(), nu / nu.sum()
    init = np.outer(mu, nu) * rng.uniform(0.0, 2.0, (n, m))
    init[rng.random((n, m)) < 0.1] = 0.0  # zeros are allowed in this geometry
    run(port, dx, dy, mu, nu, initial=np.asfortranarray(init), rho=0.5, max_iters=30,
        rel_tol=1e-30)


def test_quadratic_stop_rule_and_skinny(gpu, port):
    inst = I.config1(seed=12, n=90)
    rep, o = run(port, inst.dx, inst.dy, inst.mu, inst.nu, rho=1.0, max_iters=400, rel_tol=1e-6)
    assert rep.converged
    part = I.config3(seed=2, n=240, k=8)  # m ≤ 32: FP32 skinny chain
    run(port, part.dx, part.dy, part.mu, part.nu, rho=1.0, max_iters=30, rel_tol=1e-30)


def test_quadratic_batched_generic(gpu, port):
    # Random marginals: with uniform ones, 0/1 graphs give exactly tied
    # projection inputs, where the simplex support (and so the iterate) jumps
    # with the last bit of an fp32 iterate — not a parity-meaningful case.
    rng = np.random.default_rng(9)
    probs = []
    for k in range(2):
        p = I.config5_problem(k, seed=4)
        mu = rng.uniform(0.5, 1.5, 128)
        nu = rng.uniform(0.5, 1.5, 128)
        probs.append((p.dx, p.dy, mu / mu.sum(), nu / nu.sum()))
    cfg = gw.SolverConfig(geometry="quadratic", rho=1.0, max_iters=20, rel_tol=1e-30, quiet=True)
    reps = gw.bapg_solve_batched([gw.DistanceMatrix.trusted(p[0]) for p in probs],
                                 [gw.DistanceMatrix.trusted(p[1]) for p in probs],
                                 [gw.ProbabilityVector(p[2]) for p in probs],
                                 [gw.ProbabilityVector(p[3]) for p in probs], cfg)
    for rep, p in zip(reps, probs):
        o = port.solve(cfg.to_abi(), *p)
        assert rel(rep.final_coupling.entries(), o.final) < 1e-4
