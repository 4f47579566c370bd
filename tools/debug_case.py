import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_08115_b200 as gw
from oracle.bindings import Oracle
from tests.test_gpu_bregman import CASES
port = Oracle("port")
for name, make, over in CASES:
    if name not in ("ebpg", "hbpg"): continue
    inst = make()
    kw = dict(rel_tol=1e-30, quiet=True); kw.update(over)
    cfg = gw.SolverConfig(**kw)
    rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy), gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)
    o = port.solve(cfg.to_abi(), inst.dx, inst.dy, inst.mu, inst.nu)
    print(name, cfg, "edges", inst.dx.sum(), inst.dy.sum())
    for r, q in zip(rep.trace, o.trace):
        print(f"  it={r.iter} ph={r.phase}/{q['phase']} obj={r.objective:.9e}/{q['objective']:.9e} rel={r.rel_change:.3e}/{q['rel_change']:.3e} inf={r.marginal_infeasibility:.3e}/{q['marginal_infeasibility']:.3e}")
    f = rep.final_coupling.entries(); d = np.abs(f-o.final)
    print("  err", d.max()/np.abs(o.final).max(), np.unravel_index(np.argmax(d), d.shape))
