"""Diagnostic: one cold c4 hBPG solve through gw.solve (Python API, pageable
host arrays) with its wall time against the device trace clock; run with
GWB_PHASE_TIMES=1 for the per-phase times of the C call.

    GWB_PHASE_TIMES=1 python tools/hbpg_e2e_probe.py
"""
import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2205_08115_b200 as gw
from harness import instances as I
t=time.perf_counter(); inst = I.config4(n=20000, algorithm="hbpg"); print("instance", time.perf_counter()-t, flush=True)
s = dict(inst.solver); s.update(max_iters=200, switch_iters=100)
cfg = gw.SolverConfig(quiet=True, **s)
a = (gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy), gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu))
print("fortran", inst.dx.flags.f_contiguous, inst.dx.dtype, flush=True)
t0 = time.perf_counter(); rep = gw.solve(*a, cfg); print("wall", time.perf_counter()-t0, "device", rep.trace[-1].elapsed_seconds, flush=True)
