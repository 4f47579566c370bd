"""Golden fixtures produced by the reference's own code (tools/make_golden.py,
run where /root/reference exists).  CPU: the oracle port reproduces them.
GPU: the B200 path matches them within the north-star tolerances."""
import glob
import os

import numpy as np
import pytest

from paper_2205_08115_b200 import abi

HERE = os.path.join(os.path.dirname(__file__), "golden")
GOLD = sorted(g for g in glob.glob(os.path.join(HERE, "*.npz"))
              if not os.path.basename(g).startswith(("leaf_", "fp_")))
IDS = [os.path.basename(g)[:-4] for g in GOLD]


def residuals(z):
    """Per-record Luo-Tseng residuals (trace column 6; NaN = not recorded)."""
    tr = z["trace"]
    return tr[:, 6] if tr.shape[1] > 6 else np.full(tr.shape[0], np.nan)


def load(path):
    z = np.load(path)
    cfg = abi.Config()
    for (f, t), v in zip(abi.Config._fields_, z["config"]):
        setattr(cfg, f, float(v) if t is abi.C.c_double else int(v))
    return z, cfg


@pytest.mark.parametrize("path", GOLD, ids=IDS)
def test_port_reproduces_golden(port, path):
    z, cfg = load(path)
    r = port.solve(cfg, z["dx"], z["dy"], z["mu"], z["nu"])
    assert r.code == 0, r.message
    assert r.iterations_used == int(z["iterations"]) and r.converged == bool(z["converged"])
    assert np.abs(r.final - z["final"]).max() <= 1e-12 * np.abs(z["final"]).max()
    got = np.array([t["objective"] for t in r.trace])
    np.testing.assert_allclose(got, z["trace"][:, 1], rtol=1e-9)
    want = residuals(z)
    if not np.isnan(want).all():
        got = np.array([t["residual"] for t in r.trace])
        np.testing.assert_allclose(got, want, rtol=1e-10)


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLD, ids=IDS)
def test_gpu_matches_golden(gpu, path):
    import paper_2205_08115_b200 as gw
    z, cfg = load(path)
    names = {v: k for k, v in abi.ALGORITHMS.items()}
    sc = gw.SolverConfig(algorithm=names[cfg.algorithm], rho=cfg.rho, step=cfg.step,
                         epsilon_reg=cfg.epsilon_reg, inner_iters=cfg.inner_iters,
                         inner_tol=cfg.inner_tol, rel_tol=cfg.rel_tol, max_iters=cfg.max_iters,
                         perturbation=cfg.perturbation, switch_iters=cfg.switch_iters,
                         seed=cfg.seed, log_domain=bool(cfg.log_domain), quiet=True,
                         geometry="quadratic" if cfg.geometry == abi.QUADRATIC else "entropy",
                         record_residual=bool(cfg.record_residual))
    rep = gw.solve(gw.DistanceMatrix.trusted(z["dx"]), gw.DistanceMatrix.trusted(z["dy"]),
                   gw.ProbabilityVector(z["mu"]), gw.ProbabilityVector(z["nu"]), sc)
    final = rep.final_coupling.entries()
    assert np.abs(final - z["final"]).max() <= 1e-4 * np.abs(z["final"]).max()
    obj = rep.trace[-1].objective
    assert abs(obj - z["trace"][-1, 1]) <= 1e-5 * abs(z["trace"][-1, 1])
    if cfg.rel_tol > 1e-20 and cfg.algorithm == abi.BAPG:
        # stop-rule parity: same iteration within ±1
        assert abs(rep.iterations_used - int(z["iterations"])) <= 1
    elif cfg.rel_tol > 1e-20:
        # Bregman goldens may stop on an exact fp64 fixed point the fp32
        # iterate cannot see: never earlier than the reference.
        assert rep.iterations_used >= int(z["iterations"])
    want = residuals(z)
    if not np.isnan(want).all():
        got = np.array([r.residual for r in rep.trace])
        np.testing.assert_allclose(got, want, rtol=1e-4)


# ---- leaves: luo_tseng_residual / dykstra_project / write_coupling_csv -------

def test_port_reproduces_leaf_goldens(port):
    z = np.load(os.path.join(HERE, "leaf_residual_er40x30.npz"))
    rc, res, _ = port.luo_tseng_residual(z["dx"], z["dy"], z["pi"], z["mu"], z["nu"])
    assert rc == 0 and res == pytest.approx(float(z["residual"]), rel=1e-12)
    rc, out, _ = port.dykstra_project(z["dykstra_in"], z["mu"], z["nu"])
    assert rc == 0 and np.abs(out - z["dykstra_out"]).max() <= 1e-15
    c = np.load(os.path.join(HERE, "leaf_csv_mixed12x9.npz"))
    assert port.format_coupling_csv(c["a"]) == c["text"].tobytes()


@pytest.mark.gpu
def test_gpu_matches_leaf_goldens(gpu):
    import paper_2205_08115_b200 as gw
    z = np.load(os.path.join(HERE, "leaf_residual_er40x30.npz"))
    mu, nu = gw.ProbabilityVector(z["mu"]), gw.ProbabilityVector(z["nu"])
    res = gw.luo_tseng_residual(gw.DistanceMatrix.trusted(z["dx"]), gw.DistanceMatrix.trusted(z["dy"]),
                                z["pi"], mu, nu)
    assert abs(res - float(z["residual"])) <= 1e-4 * float(z["residual"])
    out = gw.dykstra_project(z["dykstra_in"], mu, nu)
    assert np.abs(out - z["dykstra_out"]).max() <= 1e-12 * np.abs(z["dykstra_out"]).max()
    c = np.load(os.path.join(HERE, "leaf_csv_mixed12x9.npz"))
    assert gw.format_coupling_csv(c["a"]) == c["text"].tobytes()
