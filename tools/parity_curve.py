"""Diagnostic: objective error vs iteration of the device path against a
reference fingerprint (tests/golden/fp_<case>.npz), per chain precision.

    python tools/parity_curve.py c1 auto bf16x3 3xtf32 sparse
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2205_08115_b200 as gw  # noqa: E402
from harness import cases as HC  # noqa: E402


def main():
    name, precs = sys.argv[1], sys.argv[2:] or ["auto"]
    z = np.load(os.path.join(ROOT, "tests", "golden", f"fp_{name}.npz"))
    make, over, full = HC.CASES[name]
    inst, init = make()
    ref = z["trace"][:, 1]
    for prec in precs:
        s = dict(inst.solver)
        s.update(over)
        cfg = gw.SolverConfig(quiet=True, precision=prec, **s)
        rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                       gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg,
                       gw.SolveOptions(initial=init) if init is not None else None)
        obj = np.array([r.objective for r in rep.trace])
        rel = np.abs(obj - ref[: len(obj)]) / np.abs(ref[: len(obj)])
        marks = sorted({0, 9, 99, 249, 499, 749, 999, 1249, 1499, 1749, len(obj) - 1})
        curve = " ".join(f"{k + 1}:{rel[k]:.1e}" for k in marks if k < len(obj))
        msg = f"{name} {prec}: {curve}"
        if full:
            sc = float(z["scale"])
            q = z["q"].astype(np.float64) * sc / 65535
            msg += f" | coupling err {np.abs(rep.final_coupling.entries() - q).max() / sc:.2e}"
        print(msg, flush=True)


if __name__ == "__main__":
    main()
