"""Every C-ABI leaf and the single-GPU BAPG error / observer / initial paths,
on the device, against the oracle port (oracle/gw_oracle.c, pinned to the
reference build) and the reference's own known-answer tests.

Leaves (include/gwb.h): gwb_gw_objective (solvers.cpp:64-69),
gwb_product_coupling (types.cpp:204-207), gwb_lipschitz_bound
(solvers.cpp:113-136) and the BPG step warning (:226-234), gwb_kl_scale
(projections.cpp:12-34), gwb_sinkhorn_project / _log (:92-163),
gwb_marginal_infeasibility / gwb_split_gap (diagnostics.cpp:9-27),
gwb_hard_assignment (tasks.cpp:190-200).
"""
import numpy as np
import pytest

import paper_2205_08115_b200 as gw
from harness import instances as I
from paper_2205_08115_b200 import abi

pytestmark = pytest.mark.gpu


def rng_coupling(rng, n, m, lo=0.5, hi=1.5):
    p = rng.uniform(lo, hi, (n, m))
    return np.asfortranarray(p / p.sum())


def marg(rng, n):
    v = rng.uniform(0.5, 1.5, n)
    return v / v.sum()


# ---- gw_objective ----------------------------------------------------------

def test_gw_objective_spec_kats(gpu):
    # SPEC.md:234-236
    z = gw.DistanceMatrix(np.zeros((1, 1)))
    assert gw.gw_objective(z, z, np.ones((1, 1))) == 0.0
    d = gw.DistanceMatrix(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert abs(gw.gw_objective(d, d, 0.5 * np.eye(2)) + 0.5) <= 1e-12
    assert abs(gw.gw_objective(d, d, 0.5 * np.eye(2)[::-1]) + 0.5) <= 1e-12


@pytest.mark.parametrize("kind", ["graph", "weighted"])
def test_gw_objective_vs_port(gpu, port, kind):
    rng = np.random.default_rng(3)
    if kind == "graph":
        dx = I.adjacency(300, I.erdos_renyi(300, 0.05, 1))
        dy = I.adjacency(200, I.erdos_renyi(200, 0.05, 2))
    else:
        inst = I.config2(seed=5, n=300, m=200)
        dx, dy = inst.dx, inst.dy
    pi = rng_coupling(rng, 300, 200)
    got = gw.gw_objective(gw.DistanceMatrix.trusted(dx), gw.DistanceMatrix.trusted(dy), pi)
    rc, want, st = port.gw_objective(dx, dy, pi)
    assert rc == 0
    # The leaf runs the 3xTF32 chain with an fp64 trace:
    # measured 1.5e-7 (0/1 graphs) / 1.1e-6 (weighted); bound: north star.
    assert abs(got - want) <= 1e-5 * abs(want), (got, want)


def test_gw_objective_shape_error(gpu, port):
    d = gw.DistanceMatrix(np.zeros((3, 3)))
    with pytest.raises(gw.DimensionMismatchError) as e:
        gw.gw_objective(d, d, np.ones((3, 2)) / 6)
    rc, _, st = port.gw_objective(np.zeros((3, 3)), np.zeros((3, 3)), np.ones((3, 2)) / 6)
    assert rc == abi.ERR_DIMENSION and str(e.value) == st.message.decode()


# ---- product_coupling --------------------------------------------------------

def test_product_coupling_kat_and_random(gpu, port):
    c = gw.product_coupling(gw.ProbabilityVector([0.3, 0.7]), gw.ProbabilityVector([0.5, 0.5]))
    np.testing.assert_array_equal(c.entries(), [[0.15, 0.15], [0.35, 0.35]])
    rng = np.random.default_rng(4)
    mu, nu = marg(rng, 77), marg(rng, 51)
    got = gw.product_coupling(gw.ProbabilityVector(mu), gw.ProbabilityVector(nu)).entries()
    rc, want, _ = port.product_coupling(mu, nu)
    assert rc == 0
    np.testing.assert_array_equal(got, want)  # one fp64 product per entry: bit-exact


# ---- lipschitz_bound and the BPG step warning ---------------------------------

@pytest.mark.parametrize("case", ["graphs", "gmm"])
def test_lipschitz_bound_vs_port(gpu, port, case):
    if case == "graphs":
        dx = I.adjacency(180, I.erdos_renyi(180, 0.06, 8))
        dy = I.adjacency(150, I.barabasi_albert(150, 3, 9))
    else:
        inst = I.config2(seed=6, n=160, m=120)
        dx, dy = inst.dx, inst.dy
    got = gw.lipschitz_bound(gw.DistanceMatrix.trusted(dx), gw.DistanceMatrix.trusted(dy))
    want = port.lipschitz_bound(dx, dy)
    assert abs(got - want) <= 1e-10 * want, (got, want)


def test_bpg_step_warning_text(gpu, port, capfd):
    inst = I.config1(seed=12, n=64)
    cfg = gw.SolverConfig(algorithm="bpg", step=5.0, max_iters=3, inner_iters=10,
                          rel_tol=1e-30, quiet=False)
    gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
             gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)
    err = capfd.readouterr().err
    lip = port.lipschitz_bound(inst.dx, inst.dy)
    assert 5.0 > 1.0 / lip
    want = ("bpg: step %g exceeds sigma/L_f = %g; descent is not guaranteed at this step size\n"
            % (5.0, 1.0 / lip))
    assert want in err, (err, want)


def test_bpg_no_warning_below_bound(gpu, port, capfd):
    inst = I.config1(seed=12, n=64)
    lip = port.lipschitz_bound(inst.dx, inst.dy)
    cfg = gw.SolverConfig(algorithm="bpg", step=0.5 / lip, max_iters=2, inner_iters=10,
                          rel_tol=1e-30, quiet=False)
    gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
             gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)
    assert "bpg: step" not in capfd.readouterr().err


# ---- kl_scale ------------------------------------------------------------------

@pytest.mark.parametrize("axis", [abi.ROWS, abi.COLS])
def test_kl_scale_vs_port(gpu, port, axis):
    rng = np.random.default_rng(10 + axis)
    pi = rng_coupling(rng, 90, 70)
    t = marg(rng, 90 if axis == abi.ROWS else 70)
    got = gw.kl_scale(pi, gw.ProbabilityVector(t), axis)
    rc, want, _ = port.kl_scale(pi, t, axis)
    assert rc == 0
    np.testing.assert_allclose(got, want, rtol=1e-14, atol=0)


def test_kl_scale_spec_kats(gpu):
    # SPEC.md:137-139
    np.testing.assert_allclose(gw.kl_scale(np.array([[2.0, 2.0]]), gw.ProbabilityVector([1.0]),
                                           abi.ROWS), [[0.5, 0.5]], rtol=1e-15)
    np.testing.assert_allclose(
        gw.kl_scale(np.array([[1.0, 1.0], [1.0, 3.0]]), gw.ProbabilityVector([0.5, 0.5]), abi.COLS),
        [[0.25, 0.125], [0.25, 0.375]], rtol=1e-15)


@pytest.mark.parametrize("axis,line", [(abi.ROWS, 3), (abi.COLS, 5)])
def test_kl_scale_zero_line_error(gpu, port, axis, line):
    rng = np.random.default_rng(7)
    pi = rng_coupling(rng, 8, 9)
    if axis == abi.ROWS:
        pi[line, :] = 0.0
        pi[line + 2, :] = 0.0  # the lowest offending index is reported
    else:
        pi[:, line] = 0.0
        pi[:, line + 1] = np.nan
    t = marg(rng, 8 if axis == abi.ROWS else 9)
    with pytest.raises(gw.ZeroSumLineError) as e:
        gw.kl_scale(pi, gw.ProbabilityVector(t), axis)
    rc, _, st = port.kl_scale(pi, t, axis)
    assert rc == abi.ERR_ZERO_SUM
    assert (e.value.axis, e.value.index) == (st.axis, st.index) == (axis, line)
    assert str(e.value) == st.message.decode()


# ---- sinkhorn_project / sinkhorn_project_log --------------------------------------

@pytest.mark.parametrize("log_domain", [False, True])
def test_sinkhorn_vs_port(gpu, port, log_domain):
    rng = np.random.default_rng(20 + log_domain)
    n, m = 60, 45
    mu, nu = marg(rng, n), marg(rng, m)
    k = np.asfortranarray(rng.uniform(-3, 3, (n, m)) if log_domain else rng.uniform(0.1, 2.0, (n, m)))
    fn = gw.sinkhorn_project_log if log_domain else gw.sinkhorn_project
    for tol, iters in ((1e-9, 1000), (1e-30, 7)):
        got = fn(k, gw.ProbabilityVector(mu), gw.ProbabilityVector(nu), tol, iters)
        rc, want, _ = port.sinkhorn(k, mu, nu, tol, iters, log_domain)
        assert rc == 0
        assert got.iterations == want["iterations"] and got.converged == want["converged"]
        np.testing.assert_allclose(got.coupling, want["coupling"], rtol=1e-10, atol=1e-300)
        assert abs(got.marginal_error - want["marginal_error"]) <= 1e-12


def test_sinkhorn_spec_kats(gpu):
    # kernel = μνᵀ converges in one sweep; all-ones 2×2 → 0.25.
    mu, nu = np.array([0.3, 0.7]), np.array([0.4, 0.6])
    r = gw.sinkhorn_project(np.outer(mu, nu), gw.ProbabilityVector(mu), gw.ProbabilityVector(nu),
                            1e-12, 100)
    assert r.iterations == 1 and r.converged and r.marginal_error <= 1e-15
    r = gw.sinkhorn_project(np.ones((2, 2)), gw.ProbabilityVector([0.5, 0.5]),
                            gw.ProbabilityVector([0.5, 0.5]), 1e-12, 100)
    np.testing.assert_allclose(r.coupling, 0.25, rtol=1e-15)


def test_sinkhorn_zero_sum_error(gpu, port):
    rng = np.random.default_rng(23)
    mu, nu = marg(rng, 6), marg(rng, 5)
    k = np.asfortranarray(rng.uniform(0.1, 1.0, (6, 5)))
    k[2, :] = 0.0
    with pytest.raises(gw.ZeroSumLineError) as e:
        gw.sinkhorn_project(k, gw.ProbabilityVector(mu), gw.ProbabilityVector(nu), 1e-9, 50)
    rc, _, st = port.sinkhorn(k, mu, nu, 1e-9, 50, False)
    assert rc == abi.ERR_ZERO_SUM
    assert (e.value.axis, e.value.index) == (st.axis, st.index)
    assert str(e.value) == st.message.decode()


# ---- marginal_infeasibility / split_gap / hard_assignment ------------------------

def test_diagnostics_vs_port(gpu, port):
    rng = np.random.default_rng(31)
    n, m = 120, 95
    pi, w = rng_coupling(rng, n, m), rng_coupling(rng, n, m)
    mu, nu = marg(rng, n), marg(rng, m)
    got = gw.marginal_infeasibility(pi, gw.ProbabilityVector(mu), gw.ProbabilityVector(nu))
    want = port.marginal_infeasibility(pi, mu, nu)
    assert abs(got - want) <= 1e-13 * want
    got = gw.split_gap(pi, w)
    want = port.split_gap(pi, w)
    assert abs(got - want) <= 1e-13 * want


def test_hard_assignment_ties_lowest_index(gpu, port):
    rng = np.random.default_rng(41)
    pi = np.asfortranarray(rng.integers(0, 4, (200, 37)).astype(np.float64))  # many exact ties
    got = gw.hard_assignment(pi)
    np.testing.assert_array_equal(got, port.hard_assignment(pi))
    np.testing.assert_array_equal(got, np.argmax(pi, axis=1))


# ---- single-GPU BAPG: error iteration, observer, initial coupling ------------------

def _solve(inst, **kw):
    cfg = gw.SolverConfig(quiet=True, **{**inst.solver, **kw})
    return cfg, (lambda opts=None: gw.solve(
        gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
        gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg, opts))


def _port_error(port, inst, cfg, initial=None):
    r = port.solve(cfg.to_abi(), inst.dx, inst.dy, inst.mu, inst.nu, initial=initial)
    assert r.code == abi.ERR_NUMERICAL, r.message
    return r.status


@pytest.mark.parametrize("precision", ["auto", "bf16x3", "3xtf32"])
def test_bapg_overflow_first_iteration(gpu, port, precision):
    inst = I.config1(seed=2, n=96)
    cfg, run = _solve(inst, rho=1e-6, max_iters=20, precision=precision)
    st = _port_error(port, inst, cfg)
    with pytest.raises(gw.NumericalInstabilityError) as e:
        run()
    assert (e.value.solver, e.value.iteration) == ("bapg", st.iteration) == ("bapg", 1)
    assert str(e.value) == st.message.decode() == \
        "numerical instability in bapg at iteration 1: exp overflow; increase rho"


def test_bapg_overflow_later_iteration(gpu, port):
    """The exponent max(D_X w D_Y)/ρ grows as the coupling concentrates; pick
    ρ (by the port) so the reference overflows at an iteration k > 1 with the
    same k over a ±2% band of ρ, then require the device to stop there too."""
    inst = I.config1(seed=4, n=96)
    chosen = None
    for rho in np.geomspace(1e-6, 1e-3, 60):
        its = []
        for f in (0.98, 1.0, 1.02):
            cfg, _ = _solve(inst, rho=float(rho * f), max_iters=60)
            r = port.solve(cfg.to_abi(), inst.dx, inst.dy, inst.mu, inst.nu)
            its.append(r.status.iteration if r.code == abi.ERR_NUMERICAL else 0)
        if its[0] == its[1] == its[2] and its[1] > 1:
            chosen = float(rho)
            break
    assert chosen is not None, "no stable later-iteration overflow found"
    cfg, run = _solve(inst, rho=chosen, max_iters=60)
    st = _port_error(port, inst, cfg)
    with pytest.raises(gw.NumericalInstabilityError) as e:
        run()
    assert e.value.iteration == st.iteration > 1
    assert str(e.value) == st.message.decode()


def test_bapg_nonpositive_initial_is_config_error(gpu, port):
    inst = I.config1(seed=2, n=40)
    init = np.asfortranarray(np.outer(inst.mu, inst.nu))
    init[3, 7] = 0.0
    cfg, run = _solve(inst, max_iters=5)
    with pytest.raises(gw.ConfigError) as e:
        run(gw.SolveOptions(initial=init))
    r = port.solve(cfg.to_abi(), inst.dx, inst.dy, inst.mu, inst.nu, initial=init)
    assert r.code == abi.ERR_CONFIG and str(e.value) == r.message


def test_bapg_initial_shape_error(gpu):
    inst = I.config1(seed=2, n=40)
    _, run = _solve(inst, max_iters=5)
    with pytest.raises(gw.DimensionMismatchError, match="initial coupling shape mismatch"):
        run(gw.SolveOptions(initial=np.ones((40, 39)) / 1560))


@pytest.mark.parametrize("precision", ["auto", "3xtf32"])
def test_bapg_jittered_initial_vs_port(gpu, port, precision):
    inst = I.config1(seed=9, n=200)
    init = I.jittered_product(inst.mu, inst.nu, 0.01, 99)
    cfg, run = _solve(inst, max_iters=80, precision=precision)
    rep = run(gw.SolveOptions(initial=init))
    o = port.solve(cfg.to_abi(), inst.dx, inst.dy, inst.mu, inst.nu, initial=init)
    assert o.code == 0
    err = np.abs(rep.final_coupling.entries() - o.final).max() / np.abs(o.final).max()
    assert err < 1e-4
    assert abs(rep.trace[-1].objective - o.trace[-1]["objective"]) <= 1e-5 * abs(o.trace[-1]["objective"])


@pytest.mark.parametrize("algorithm", ["bapg", "hbpg"])
def test_observer_sees_every_iteration(gpu, port, algorithm):
    """SolveOptions::observer (solvers.hpp:42-44): called after every outer
    iteration with the current iterate (solvers.cpp:206, 282, 352; hBPG
    phase 2 shifted by the phase-1 count, :408-413); the iterate it sees at
    iteration k equals the port's iterate after k iterations."""
    inst = I.config1(seed=14, n=64)
    extra = dict(epsilon_reg=0.1, step=5.0, inner_iters=10, switch_iters=3) if algorithm == "hbpg" else {}
    cfg, run = _solve(inst, algorithm=algorithm, max_iters=6, rel_tol=1e-30, **extra)
    seen = []

    def obs(it, pi, w):
        seen.append((it, np.array(pi, copy=True), None if w is None else np.array(w, copy=True)))

    rep = run(gw.SolveOptions(observer=obs))
    assert [s[0] for s in seen] == list(range(1, rep.iterations_used + 1)) == list(range(1, 7))
    assert all((s[2] is not None) == (algorithm == "bapg") for s in seen)
    for k in (1, 3, 6):
        c = cfg.to_abi()
        c.max_iters = k
        o = port.solve(c, inst.dx, inst.dy, inst.mu, inst.nu)
        want = o.pi if algorithm == "bapg" else o.final
        got = seen[k - 1][1]
        assert np.abs(got - want).max() <= 1e-4 * np.abs(want).max(), k
        if algorithm == "bapg":
            assert np.abs(seen[k - 1][2] - o.w).max() <= 1e-4 * np.abs(o.w).max()


def test_observer_exception_aborts(gpu):
    inst = I.config1(seed=14, n=48)
    _, run = _solve(inst, max_iters=10, rel_tol=1e-30)
    calls = []

    def obs(it, pi, w):
        calls.append(it)
        if it == 2:
            raise KeyError("stop")

    with pytest.raises(KeyError, match="stop"):
        run(gw.SolveOptions(observer=obs))
    assert calls == [1, 2]
