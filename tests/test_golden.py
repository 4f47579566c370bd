"""Golden fixtures produced by the reference's own code (tools/make_golden.py,
run where /root/reference exists).  CPU: the oracle port reproduces them.
GPU: the B200 path matches them within the north-star tolerances."""
import glob
import os

import numpy as np
import pytest

from paper_2205_08115_b200 import abi

GOLD = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
IDS = [os.path.basename(g)[:-4] for g in GOLD]


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
                         seed=cfg.seed, log_domain=bool(cfg.log_domain), quiet=True)
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
