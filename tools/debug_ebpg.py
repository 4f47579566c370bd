import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_08115_b200 as gw
from paper_2205_08115_b200 import instances as I
from oracle.bindings import Oracle
port = Oracle("port")
inst = I.config1(seed=5, n=128)
for iters in (1, 2, 4, 12):
  for inner in (1, 3, 10):
    for logd in (False, True):
        cfg = gw.SolverConfig(algorithm="ebpg", epsilon_reg=0.1, max_iters=iters, inner_iters=inner, rel_tol=1e-30, quiet=True, log_domain=logd)
        rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy), gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)
        o = port.solve(cfg.to_abi(), inst.dx, inst.dy, inst.mu, inst.nu)
        f = rep.final_coupling.entries(); d = np.abs(f - o.final); i, j = np.unravel_index(np.argmax(d), d.shape)
        print(f"iters={iters} inner={inner} log={logd} err={d.max()/np.abs(o.final).max():.2e} at ({i},{j}) ours={f[i,j]:.6e} ref={o.final[i,j]:.6e} rowsum_ours={f[i].sum():.6e} ref={o.final[i].sum():.6e}")
