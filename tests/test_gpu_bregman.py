"""eBPG / BPG / hBPG on the device vs the CPU oracle (solvers.cpp:219-426):
final coupling within 1e-4 of its scale, objective within 1e-5, trace
phases/iterations identical, error semantics identical."""
import glob
import os

import numpy as np
import pytest

import paper_2205_08115_b200 as gw
from paper_2205_08115_b200 import abi
from harness import instances as I

pytestmark = pytest.mark.gpu

CASES = [
    ("ebpg", lambda: I.config1(seed=5, n=128), dict(algorithm="ebpg", epsilon_reg=0.1, max_iters=12, inner_iters=10)),
    ("ebpg-log", lambda: I.config1(seed=6, n=96), dict(algorithm="ebpg", epsilon_reg=0.01, log_domain=True, max_iters=8, inner_iters=20)),
    ("bpg", lambda: I.config1(seed=7, n=128), dict(algorithm="bpg", step=5.0, max_iters=10, inner_iters=10)),
    ("bpg-perturb", lambda: I.config1(seed=9, n=64), dict(algorithm="bpg", perturbation=0.01, max_iters=8, inner_iters=20)),
    ("hbpg", lambda: I.config1(seed=8, n=128), dict(algorithm="hbpg", epsilon_reg=0.1, step=5.0, inner_iters=10, switch_iters=6, max_iters=14)),
    ("hbpg-gmm", lambda: I.config2(seed=3, n=160, m=128), dict(algorithm="hbpg", epsilon_reg=0.1, step=1.0, inner_iters=10, switch_iters=4, max_iters=8)),
    ("ebpg-stop", lambda: I.config1(seed=10, n=64), dict(algorithm="ebpg", epsilon_reg=0.1, max_iters=200, inner_iters=50, rel_tol=1e-6)),
]


@pytest.mark.parametrize("name,make,over", CASES, ids=[c[0] for c in CASES])
def test_bregman_parity(gpu, port, name, make, over):
    inst = make()
    kw = dict(rel_tol=1e-30, quiet=True)
    kw.update(over)
    cfg = gw.SolverConfig(**kw)
    rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                   gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)
    o = port.solve(cfg.to_abi(), inst.dx, inst.dy, inst.mu, inst.nu)
    assert o.code == 0, o.message
    assert rep.iterations_used == o.iterations_used
    assert rep.converged == o.converged
    f, fr = rep.final_coupling.entries(), o.final
    assert np.abs(f - fr).max() <= 1e-4 * np.abs(fr).max()
    assert [t.phase for t in rep.trace] == [t["phase"] for t in o.trace]
    obj, obj_ref = rep.trace[-1].objective, o.trace[-1]["objective"]
    assert abs(obj - obj_ref) <= 1e-5 * abs(obj_ref)
    for r, q in zip(rep.trace, o.trace):
        assert abs(r.objective - q["objective"]) <= 1e-4 * abs(q["objective"])


@pytest.mark.parametrize("over,solver", [
    (dict(algorithm="bpg", step=1e7, inner_iters=5), "bpg"),
    (dict(algorithm="ebpg", epsilon_reg=1e-5, inner_iters=5), "ebpg"),
])
def test_bregman_errors(gpu, port, over, solver):
    inst = I.config1(seed=2, n=48)
    cfg = gw.SolverConfig(rel_tol=1e-30, max_iters=5, quiet=True, **over)
    o = port.solve(cfg.to_abi(), inst.dx, inst.dy, inst.mu, inst.nu)
    with pytest.raises(gw.NumericalInstabilityError) as ei:
        gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                 gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)
    assert str(ei.value) == o.message
    assert ei.value.solver == solver


GOLD = sorted(g for g in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*bpg*.npz"))
              if not os.path.basename(g).startswith("fp_"))


@pytest.mark.parametrize("path", GOLD, ids=[os.path.basename(g)[:-4] for g in GOLD])
def test_bregman_golden(gpu, path):
    from tests.test_golden import load
    z, cfg = load(path)
    names = {abi.EBPG: "ebpg", abi.BPG: "bpg", abi.HBPG: "hbpg"}
    sc = gw.SolverConfig(algorithm=names[cfg.algorithm], epsilon_reg=cfg.epsilon_reg, step=cfg.step,
                         inner_iters=cfg.inner_iters, inner_tol=cfg.inner_tol,
                         switch_iters=cfg.switch_iters, max_iters=cfg.max_iters,
                         rel_tol=cfg.rel_tol, quiet=True)
    rep = gw.solve(gw.DistanceMatrix.trusted(z["dx"]), gw.DistanceMatrix.trusted(z["dy"]),
                   gw.ProbabilityVector(z["mu"]), gw.ProbabilityVector(z["nu"]), sc)
    if bool(z["converged"]) and z["trace"][-1, 4] == 0.0:
        # The fp64 reference stopped on an exactly stationary iterate
        # (rel_change == 0 ≤ rel_tol); fp32 iterates keep ~1e-8 noise, so
        # the GPU runs on (to max_iters) at the same fixed point.
        assert rep.iterations_used >= int(z["iterations"])
    else:
        assert rep.iterations_used == int(z["iterations"])
    assert np.abs(rep.final_coupling.entries() - z["final"]).max() <= 1e-4 * np.abs(z["final"]).max()
    assert abs(rep.trace[-1].objective - z["trace"][-1, 1]) <= 1e-5 * abs(z["trace"][-1, 1])


@pytest.mark.parametrize("precision", ["auto", "bf16x3"])
def test_hbpg_initial_coupling_and_precisions(gpu, port, precision):
    # AUTO runs the Bregman chain as f16x2 for 0/1 graphs; an initial
    # coupling concentrated on a permutation (entries 0.9/n ≫ μ_i ν_j) sets
    # the f16x2 iterate bound.
    inst = I.config1(seed=12, n=200)
    n = inst.dx.shape[0]
    rng = np.random.default_rng(3)
    init = np.full((n, n), 0.1 / (n * n))
    init[np.arange(n), rng.permutation(n)] += 0.9 / n
    init = np.asfortranarray(init / init.sum())
    cfg = gw.SolverConfig(algorithm="hbpg", epsilon_reg=0.1, step=5.0, inner_iters=10,
                          switch_iters=5, max_iters=10, rel_tol=1e-30, quiet=True,
                          precision=precision)
    rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                   gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg,
                   gw.SolveOptions(initial=init))
    o = port.solve(cfg.to_abi(), inst.dx, inst.dy, inst.mu, inst.nu, init)
    assert o.code == 0, o.message
    assert rep.iterations_used == o.iterations_used
    f, fr = rep.final_coupling.entries(), o.final
    assert np.abs(f - fr).max() <= 1e-4 * np.abs(fr).max()
    for r, q in zip(rep.trace, o.trace):
        assert abs(r.objective - q["objective"]) <= 1e-5 * abs(q["objective"])
