"""c4 hBPG rate through the public gw.solve call (host fp64 in/out).

Per-iteration time is taken from the device-side `elapsed_seconds` trace
(globaltimer since reset) so the host↔device copies of the 3.2 GB inputs do
not pollute it; the whole call's wall time is reported next to it.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2205_08115_b200 as gw
from harness import instances as I


def run(n, iters, switch):
    inst = I.config4(n=n, algorithm="hbpg")
    s = dict(inst.solver)
    s.update(max_iters=iters, switch_iters=switch)
    cfg = gw.SolverConfig(quiet=True, **s)
    args = (gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
            gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu))
    t0 = time.perf_counter()
    rep = gw.solve(*args, cfg)
    wall = time.perf_counter() - t0
    tr = rep.trace
    ph1 = [r for r in tr if r.phase == 1]
    ph2 = [r for r in tr if r.phase == 2]

    def rate(rs):
        if len(rs) < 2:
            return None
        return (len(rs) - 1) / (rs[-1].elapsed_seconds - rs[0].elapsed_seconds)

    return {"n": n, "iters": rep.iterations_used, "wall_s": wall,
            "ebpg_it_per_s": rate(ph1), "bpg_it_per_s": rate(ph2),
            "device_s": tr[-1].elapsed_seconds if tr else None,
            "objective": tr[-1].objective if tr else None,
            "phases": sorted({r.phase for r in tr})}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=20000)
    ap.add_argument("--iters", type=int, default=12)
    ap.add_argument("--switch", type=int, default=6)
    a = ap.parse_args()
    print(json.dumps(run(a.size, a.iters, a.switch)), flush=True)
