"""Dykstra projection / Luo-Tseng residual throughput on the device
(csrc/residual.cu).  Prints one JSON line per size: sweeps, device ms for
the sweep loop, ms per sweep and the algorithmic HBM rate of a sweep
(64 B per element: the row pass reads x, p and writes y, p; the column pass
reads y, q and writes x, q; all fp64)."""
import ctypes as C
import json
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2205_08115_b200 as gw  # noqa: E402
from paper_2205_08115_b200 import abi
from harness import instances as I  # noqa: E402


def stats():
    sw, ms = C.c_int32(0), C.c_double(0)
    abi.load().gwb_dykstra_last_stats(C.byref(sw), C.byref(ms))
    return sw.value, ms.value


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [1024, 4096, 8192]
    for n in sizes:
        rng = np.random.default_rng(n)
        mu = rng.uniform(0.5, 1.5, n)
        nu = rng.uniform(0.5, 1.5, n)
        mu, nu = mu / mu.sum(), nu / nu.sum()
        pi = np.asfortranarray(np.outer(mu, nu) * rng.uniform(0.0, 3.0, (n, n)))
        t = time.perf_counter()
        gw.dykstra_project(pi, gw.ProbabilityVector(mu), gw.ProbabilityVector(nu))
        wall = time.perf_counter() - t
        sw, ms = stats()
        per = ms / max(sw, 1)
        line = dict(kind="dykstra", n=n, m=n, sweeps=sw, loop_ms=round(ms, 3),
                    ms_per_sweep=round(per, 4), gbs=round(64.0 * n * n / (per * 1e-3) / 1e9, 1),
                    wall_s=round(wall, 3))
        print(json.dumps(line), flush=True)
    # A residual on a BA alignment instance (the readout's use).
    n = sizes[-1]
    inst = I.config1(seed=1, n=n)
    plan = np.asfortranarray(np.outer(inst.mu, inst.nu))
    t = time.perf_counter()
    r = gw.luo_tseng_residual(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                              plan, gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu))
    wall = time.perf_counter() - t
    sw, ms = stats()
    print(json.dumps(dict(kind="residual", n=n, residual=r, sweeps=sw, loop_ms=round(ms, 3),
                          ms_per_sweep=round(ms / max(sw, 1), 4), wall_s=round(wall, 3))), flush=True)


if __name__ == "__main__":
    main()
