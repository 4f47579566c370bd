"""Stop-rule behaviour of quadratic-geometry BAPG across chain precisions
(diagnostic): iterations used by the device path vs the oracle, uniform
marginals (exactly tied projection inputs) and random ones."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2205_08115_b200 as gw
from harness import instances as I
from oracle.bindings import Oracle

port = Oracle("port")
inst = I.config1(seed=12, n=90)
rng = np.random.default_rng(21)
mu_r = rng.uniform(0.5, 1.5, 90)
nu_r = rng.uniform(0.5, 1.5, 90)
for label, mu, nu in [("uniform", inst.mu, inst.nu), ("random", mu_r / mu_r.sum(), nu_r / nu_r.sum())]:
    for prec in ["auto", "bf16x3", "3xtf32", "bf16x2"]:
        cfg = gw.SolverConfig(geometry="quadratic", quiet=True, rho=1.0, max_iters=400, rel_tol=1e-6,
                              precision=prec)
        rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                       gw.ProbabilityVector(mu), gw.ProbabilityVector(nu), cfg)
        o = port.solve(cfg.to_abi(), inst.dx, inst.dy, mu, nu)
        err = np.abs(rep.final_coupling.entries() - o.final).max() / np.abs(o.final).max()
        print(os.environ.get("GWB_GEMM_UNFUSED", "fused"), label, prec, rep.iterations_used,
              o.iterations_used, f"{err:.2e}", flush=True)
