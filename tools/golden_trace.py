"""Diagnostic: per-record objective of the device path against a golden
fixture (tests/golden/<name>.npz), for the given chain precisions."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2205_08115_b200 as gw  # noqa: E402
from tests.test_golden import load  # noqa: E402
from paper_2205_08115_b200 import abi  # noqa: E402

name, precs = sys.argv[1], sys.argv[2:] or ["auto"]
z, cfg = load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
names = {v: k for k, v in abi.ALGORITHMS.items()}
for prec in precs:
    sc = gw.SolverConfig(algorithm=names[cfg.algorithm], rho=cfg.rho, step=cfg.step,
                         epsilon_reg=cfg.epsilon_reg, inner_iters=cfg.inner_iters,
                         inner_tol=cfg.inner_tol, rel_tol=cfg.rel_tol, max_iters=cfg.max_iters,
                         perturbation=cfg.perturbation, switch_iters=cfg.switch_iters,
                         seed=cfg.seed, log_domain=bool(cfg.log_domain), quiet=True,
                         geometry="quadratic" if cfg.geometry == abi.QUADRATIC else "entropy",
                         precision=prec)
    rep = gw.solve(gw.DistanceMatrix.trusted(z["dx"]), gw.DistanceMatrix.trusted(z["dy"]),
                   gw.ProbabilityVector(z["mu"]), gw.ProbabilityVector(z["nu"]), sc)
    obj = np.array([r.objective for r in rep.trace])
    ref = z["trace"][: len(obj), 1]
    print(name, prec, " ".join(f"{k + 1}:{abs(a - b) / abs(b):.1e}" for k, (a, b) in enumerate(zip(obj, ref))))
