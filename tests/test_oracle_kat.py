"""Known-answer tests of the CPU oracle, from the reference's own tests
(proj/tests/test_core.cpp) and the SPEC.md prose KATs.
Each runs against the C restatement ("port") and, when built, the
reference's own TUs ("reference") — pinning the restatement."""
import numpy as np
import pytest

from paper_2205_08115_b200 import abi
from tests.conftest import have_ref

KINDS = ["port"] + (["reference"] if have_ref() else [])


@pytest.fixture(params=KINDS, scope="module")
def orc(request):
    from oracle.bindings import Oracle
    return Oracle(request.param)


def cfg(**kw):
    return abi.default_config(quiet=1, **kw)


# --- product_coupling: test_core.cpp:56-89, SPEC.md:92-94 ------------------
def test_product_coupling_values(orc):
    rc, p, _ = orc.product_coupling([1.0], [1.0])
    assert rc == 0 and p[0, 0] == 1.0
    rc, p, _ = orc.product_coupling([0.5, 0.5], [0.5, 0.5])
    assert np.all(p == 0.25)
    rc, p, _ = orc.product_coupling([0.3, 0.7], [0.5, 0.5])
    np.testing.assert_allclose(p, [[0.15, 0.15], [0.35, 0.35]], rtol=1e-14)


def test_product_coupling_marginals(orc):
    rng = np.random.default_rng(7)
    for trial in range(50):
        n, m = 2 + trial % 6, 2 + (trial // 2) % 6
        a = 0.2 + rng.random(n)
        b = 0.2 + rng.random(m)
        a /= a.sum()
        b /= b.sum()
        _, p, _ = orc.product_coupling(a, b)
        assert np.abs(p.sum(axis=1) - a).max() <= 1e-15
        assert np.abs(p.sum(axis=0) - b).max() <= 1e-15


# --- gw_objective: SPEC.md:234-236, oracles.hpp:54-72 ----------------------
def quadruple_loop(dx, dy, pi, w):
    return -np.einsum("ik,jl,ij,kl->", dx, dy, pi, w)


def test_gw_objective_kats(orc):
    assert orc.gw_objective([[0.0]], [[0.0]], [[1.0]])[1] == 0.0
    d = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert orc.gw_objective(d, d, 0.5 * np.eye(2))[1] == pytest.approx(-0.5, abs=1e-15)
    assert orc.gw_objective(d, d, 0.5 * np.eye(2)[::-1])[1] == pytest.approx(-0.5, abs=1e-15)


def test_gw_objective_vs_quadruple_loop(orc):
    rng = np.random.default_rng(3)
    for n, m in [(3, 4), (5, 2), (4, 4)]:
        a = rng.random((n, n)); dx = a + a.T
        b = rng.random((m, m)); dy = b + b.T
        pi = rng.random((n, m)); pi /= pi.sum()
        got = orc.gw_objective(dx, dy, pi)[1]
        assert got == pytest.approx(quadruple_loop(dx, dy, pi, pi), rel=1e-12)


def test_gw_objective_shape_error(orc):
    rc, _, st = orc.gw_objective(np.zeros((2, 2)), np.zeros((3, 3)), np.zeros((3, 2)))
    assert rc == abi.ERR_DIMENSION
    assert st.message.decode() == "gw_objective: coupling shape mismatch"


# --- kl_scale: SPEC.md:137-139, projections.cpp:12-34 ----------------------
def test_kl_scale_kats(orc):
    rc, out, _ = orc.kl_scale([[2.0, 2.0]], [1.0], abi.ROWS)
    np.testing.assert_allclose(out, [[0.5, 0.5]])
    rc, out, _ = orc.kl_scale([[1.0, 1.0], [1.0, 3.0]], [0.5, 0.5], abi.COLS)
    np.testing.assert_allclose(out, [[0.25, 0.125], [0.25, 0.375]], rtol=1e-15)


def test_kl_scale_idempotent_and_zero_line(orc):
    rng = np.random.default_rng(1)
    pi = 0.1 + rng.random((4, 5))
    mu = np.full(4, 0.25)
    _, a, _ = orc.kl_scale(pi, mu, abi.ROWS)
    _, b, _ = orc.kl_scale(a, mu, abi.ROWS)
    assert np.abs(a - b).max() <= 1e-14
    z = pi.copy(); z[2, :] = 0.0
    rc, _, st = orc.kl_scale(z, mu, abi.ROWS)
    assert rc == abi.ERR_ZERO_SUM and st.index == 2
    assert st.message.decode() == "row 2 has nonpositive sum; cannot rescale"
    z = pi.copy(); z[:, 3] = 0.0
    rc, _, st = orc.kl_scale(z, np.full(5, 0.2), abi.COLS)
    assert st.message.decode() == "column 3 has nonpositive sum; cannot rescale"


# --- Sinkhorn: SPEC.md:167-169, oracles.hpp:213-224 -------------------------
def over_iterated(k, mu, nu, sweeps):
    k = np.array(k, dtype=float)
    for _ in range(sweeps):
        k *= (mu / k.sum(axis=1))[:, None]
        k *= (nu / k.sum(axis=0))[None, :]
    return k


def test_sinkhorn_kats(orc):
    mu, nu = np.array([0.3, 0.7]), np.array([0.4, 0.6])
    rc, r, _ = orc.sinkhorn(np.outer(mu, nu), mu, nu, 1e-15, 10)
    assert r["iterations"] == 1 and r["marginal_error"] <= 1e-15
    u = np.array([0.5, 0.5])
    rc, r, _ = orc.sinkhorn(np.ones((2, 2)), u, u, 1e-12, 100)
    np.testing.assert_allclose(r["coupling"], 0.25)
    k = np.array([[1.0, 2.0], [3.0, 1.0]])
    rc, r, _ = orc.sinkhorn(k, u, u, 1e-10, 100000)
    assert r["converged"]
    np.testing.assert_allclose(r["coupling"], over_iterated(k, u, u, 100000), atol=1e-9)


def test_sinkhorn_log_matches_plain(orc):
    rng = np.random.default_rng(4)
    e = rng.normal(size=(6, 5))
    mu = np.full(6, 1 / 6)
    nu = np.full(5, 0.2)
    _, a, _ = orc.sinkhorn(np.exp(e), mu, nu, 1e-12, 500)
    _, b, _ = orc.sinkhorn(e, mu, nu, 1e-12, 500, log_domain=True)
    np.testing.assert_allclose(a["coupling"], b["coupling"], atol=1e-12)


# --- solvers: SPEC.md:273-306 ------------------------------------------------
def test_bapg_single_point(orc):
    r = orc.solve(cfg(max_iters=5), [[0.0]], [[0.0]], [1.0], [1.0])
    assert r.code == 0
    assert r.final[0, 0] == 1.0 and r.pi[0, 0] == 1.0 and r.w[0, 0] == 1.0


@pytest.mark.parametrize("algo", [abi.BAPG, abi.EBPG, abi.BPG, abi.HBPG])
def test_zero_distance_keeps_product_coupling(orc, algo):
    mu = np.array([0.2, 0.3, 0.5])
    nu = np.array([0.6, 0.4])
    r = orc.solve(cfg(algorithm=algo, max_iters=7, rel_tol=1e-30, switch_iters=3, inner_iters=50),
                  np.zeros((3, 3)), np.zeros((2, 2)), mu, nu)
    assert r.code == 0, r.message
    np.testing.assert_allclose(r.final, np.outer(mu, nu), atol=1e-15)


def test_bapg_split_gap_decreases_with_rho(orc):
    rng = np.random.default_rng(11)
    a = rng.random((5, 5)); dx = a + a.T
    b = rng.random((5, 5)); dy = b + b.T
    u = np.full(5, 0.2)
    gaps = []
    for rho in (0.1, 0.2, 0.4, 0.8):
        r = orc.solve(cfg(rho=rho, max_iters=2000), dx, dy, u, u)
        assert r.code == 0, r.message
        gaps.append(r.trace[-1]["split_gap"])
    assert all(x > y for x, y in zip(gaps, gaps[1:])), gaps
    slope = np.polyfit(np.log([0.1, 0.2, 0.4, 0.8]), np.log(gaps), 1)[0]
    assert -1.5 <= slope <= -0.5, slope


def test_bapg_halves_feasible(orc):
    rng = np.random.default_rng(2)
    a = rng.random((6, 6)); dx = a + a.T
    b = rng.random((4, 4)); dy = b + b.T
    mu = 0.2 + rng.random(6); mu /= mu.sum()
    nu = 0.2 + rng.random(4); nu /= nu.sum()
    r = orc.solve(cfg(rho=0.5, max_iters=30, rel_tol=1e-30), dx, dy, mu, nu)
    assert np.abs(r.pi.sum(axis=1) - mu).max() <= 1e-12
    assert np.abs(r.w.sum(axis=0) - nu).max() <= 1e-12


def test_hbpg_degenerate_phases(orc):
    rng = np.random.default_rng(5)
    a = rng.random((5, 5)); dx = a + a.T
    u = np.full(5, 0.2)
    common = dict(max_iters=6, rel_tol=1e-30, inner_iters=50, step=0.05, epsilon_reg=1.0)
    h0 = orc.solve(cfg(algorithm=abi.HBPG, switch_iters=0, **common), dx, dx, u, u)
    b = orc.solve(cfg(algorithm=abi.BPG, **common), dx, dx, u, u)
    np.testing.assert_array_equal(h0.final, b.final)
    assert [t["phase"] for t in h0.trace] == [2] * 6
    hm = orc.solve(cfg(algorithm=abi.HBPG, switch_iters=6, **common), dx, dx, u, u)
    e = orc.solve(cfg(algorithm=abi.EBPG, **common), dx, dx, u, u)
    np.testing.assert_array_equal(hm.final, e.final)
    assert [t["phase"] for t in hm.trace] == [1] * 6
    h3 = orc.solve(cfg(algorithm=abi.HBPG, switch_iters=3, **common), dx, dx, u, u)
    assert [t["iter"] for t in h3.trace] == list(range(1, 7))
    assert [t["phase"] for t in h3.trace] == [1, 1, 1, 2, 2, 2]


def test_overflow_error_format(orc):
    d = np.array([[0.0, 1.0], [1.0, 0.0]])
    u = np.array([0.5, 0.5])
    r = orc.solve(cfg(rho=1e-5, max_iters=3), d, d, u, u)
    assert r.code == abi.ERR_NUMERICAL
    assert r.message == "numerical instability in bapg at iteration 1: exp overflow; increase rho"
    assert r.status.solver == b"bapg" and r.status.iteration == 1


def test_config_validation(orc):
    for field, val, msg in [("rho", 0.0, "rho must be positive"),
                            ("max_iters", 0, "max-iters must be >= 1"),
                            ("perturbation", 1.0, "perturbation must lie in [0, 1)"),
                            ("switch_iters", -1, "switch-iters must be >= 0")]:
        r = orc.solve(cfg(**{field: val}), [[0.0]], [[0.0]], [1.0], [1.0])
        assert r.code == abi.ERR_CONFIG and r.message == msg


# --- lipschitz_bound: SPEC lipschitz KATs, oracles.hpp:187-208 ---------------
def test_lipschitz(orc):
    z = np.zeros((3, 3))
    assert orc.lipschitz_bound(z, z) == 0.0
    d = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert orc.lipschitz_bound(d, d) == pytest.approx(1.0, rel=1e-10)
    rng = np.random.default_rng(9)
    a = rng.random((5, 5)); a = a + a.T
    b = rng.random((4, 4)); b = b + b.T
    exp = np.abs(np.linalg.eigvalsh(a)).max() * np.abs(np.linalg.eigvalsh(b)).max()
    assert orc.lipschitz_bound(a, b) == pytest.approx(exp, rel=1e-8)


def test_hard_assignment_ties(orc):
    pi = np.array([[0.1, 0.3, 0.3], [0.2, 0.1, 0.0], [0.0, 0.0, 0.0]])
    np.testing.assert_array_equal(orc.hard_assignment(pi), [1, 0, 0])
