"""Diagnostic: per-problem objective error of the on-chip batched kernel
against the c5 reference fingerprint (tests/golden/fp_c5.npz): worst
record, where it sits, and the stop iterations.

    python tools/c5_diag.py [count]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2205_08115_b200 as gw  # noqa: E402
from harness import instances as I  # noqa: E402


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    z = np.load(os.path.join(ROOT, "tests", "golden", "fp_c5.npz"))
    insts = [I.config5_problem(k) for k in range(count)]
    cfg = gw.SolverConfig(quiet=True, **insts[0].solver)
    reps = gw.bapg_solve_batched([gw.DistanceMatrix.trusted(i.dx) for i in insts],
                                 [gw.DistanceMatrix.trusted(i.dy) for i in insts],
                                 [gw.ProbabilityVector(i.mu) for i in insts],
                                 [gw.ProbabilityVector(i.nu) for i in insts], cfg)
    rows = []
    for k, rep in enumerate(reps):
        ref_it = int(z["iterations"][k])
        obj = np.array([r.objective for r in rep.trace])[:ref_it]
        want = z["objective"][k][: len(obj)]
        rel = np.abs(obj - want) / np.abs(want).max()
        at = int(rel.argmax())
        rows.append((rel.max(), k, at, rep.iterations_used, ref_it, rel[0], rel[min(9, len(rel) - 1)]))
    rows.sort(reverse=True)
    for r in rows[:12]:
        print("err %.2e problem %3d at record %3d (used %d, ref %d); rec1 %.1e rec10 %.1e" % r)
    errs = np.array([r[0] for r in rows])
    print(f"median {np.median(errs):.2e}, mean {errs.mean():.2e}, max {errs.max():.2e}")


if __name__ == "__main__":
    main()
