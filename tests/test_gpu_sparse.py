"""Sparse chain (precision "sparse", csrc/sparse.cu): the D_X·π·D_Y chain as
two CSR row-gathers with fp32 exact-order sums.  Same parity bar as the
dense chains against the CPU oracle (π 1e-4 relative to scale, objective
1e-5 relative), on 0/1 graphs, ragged shapes and weighted (dense-pattern)
structure matrices."""
import numpy as np
import pytest

import paper_2205_08115_b200 as gw
from harness import instances as I

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def run(port, dx, dy, mu, nu, **solver):
    cfg = gw.SolverConfig(precision="sparse", quiet=True, **solver)
    rep = gw.solve(gw.DistanceMatrix.trusted(dx), gw.DistanceMatrix.trusted(dy),
                   gw.ProbabilityVector(mu), gw.ProbabilityVector(nu), cfg)
    o = port.solve(cfg.to_abi(), dx, dy, mu, nu)
    assert o.code == 0, o.message
    assert rep.iterations_used == o.iterations_used
    assert rel(rep.final_coupling.entries(), o.final) < 1e-4
    assert rel(rep.pi_half.entries(), o.pi) < 1e-4
    assert rel(rep.w_half.entries(), o.w) < 1e-4
    for r, q in zip(rep.trace, o.trace):
        assert abs(r.objective - q["objective"]) <= 1e-5 * abs(q["objective"])
        assert abs(r.rel_change - q["rel_change"]) <= 1e-3 * q["rel_change"] + 1e-7
    return rep, o


def test_sparse_er_alignment(gpu, port):
    inst = I.config1(seed=6, n=400)
    run(port, inst.dx, inst.dy, inst.mu, inst.nu, rho=0.1, max_iters=80, rel_tol=1e-30)


def test_sparse_ba_alignment_converges(gpu, port):
    inst = I.config4(n=600)
    rep, o = run(port, inst.dx, inst.dy, inst.mu, inst.nu, rho=0.1, max_iters=300, rel_tol=1e-5)
    assert rep.converged == bool(o.converged)


def test_sparse_ragged_nonuniform(gpu, port):
    rng = np.random.default_rng(3)
    n, m = 203, 150
    dx = I.adjacency(n, I.erdos_renyi(n, 0.05, 11))
    dy = I.adjacency(m, I.erdos_renyi(m, 0.07, 12))
    mu = rng.uniform(0.5, 1.5, n)
    nu = rng.uniform(0.5, 1.5, m)
    run(port, dx, dy, mu / mu.sum(), nu / nu.sum(), rho=0.05, max_iters=60, rel_tol=1e-30)


def test_sparse_weighted_dense_pattern(gpu, port):
    # Euclidean distances: every off-diagonal entry is stored (nnz ≈ n²).
    g = I.config2(seed=2, n=96, m=72)
    run(port, g.dx, g.dy, g.mu, g.nu, rho=0.05, max_iters=40, rel_tol=1e-30)


def test_sparse_graph_inputs_match_dense_inputs(gpu):
    inst = I.config1(seed=8, n=256)
    e = I.erdos_renyi(256, 0.01, 8)
    cfg = gw.SolverConfig(precision="sparse", rho=0.1, max_iters=30, rel_tol=1e-30, quiet=True)
    u = gw.ProbabilityVector(inst.mu)
    gx = gw.Graph(256, e)
    a = gw.solve(gw.adjacency_distance(gx), gw.adjacency_distance(gx), u, u, cfg)
    d = gw.adjacency_distance(gx).entries()
    b = gw.solve(gw.DistanceMatrix(d), gw.DistanceMatrix(d), u, u, cfg)
    assert np.array_equal(a.final_coupling.entries(), b.final_coupling.entries())
