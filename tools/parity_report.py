"""Print GPU-vs-oracle parity numbers for small instances (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_08115_b200 as gw
from harness import instances as I
from oracle.bindings import Oracle

port = Oracle("port")
cases = [("c1-256", I.config1(seed=3, n=256), 60), ("c1-1000", I.config1(seed=0), 100),
         ("c2-320x256", I.config2(seed=1, n=320, m=256), 40), ("c3-800", I.config3(seed=0, n=800), 100)]
for name, inst, iters in cases:
    o = port.solve(gw.SolverConfig(quiet=True, **{**inst.solver, "max_iters": iters}).to_abi(),
                   inst.dx, inst.dy, inst.mu, inst.nu)
    for prec in sys.argv[1].split(",") if len(sys.argv) > 1 else ("tf32", "3xtf32", "bf16x3", "bf16x2", "f16x2"):
        cfg = gw.SolverConfig(precision=prec, quiet=True, **{**inst.solver, "max_iters": iters})
        t = time.time()
        rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                       gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)
        dt = time.time() - t
        pe = np.abs(rep.final_coupling.entries() - o.final).max() / np.abs(o.final).max()
        oe = abs(rep.trace[-1].objective - o.trace[-1]["objective"]) / abs(o.trace[-1]["objective"])
        am = np.mean(gw.hard_assignment(rep.final_coupling.entries()) == np.argmax(o.final, axis=1))
        re = max(abs(r.rel_change - q["rel_change"]) / q["rel_change"] for r, q in zip(rep.trace, o.trace))
        print(f"{name:12s} {prec:7s} pi_err={pe:.2e} obj_err={oe:.2e} argmax_eq={am:.4f} relchg_err={re:.1e} t={dt:.2f}s obj={o.trace[-1]['objective']:.6e}")
