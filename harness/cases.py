"""The seeded BASELINE.json cases shared by tools/make_fingerprints.py (which
runs the reference build on them, here) and the GPU parity tests (which
regenerate them on the box and compare against the committed fingerprints,
tests/golden/fp_*.npz).  Bench / test harness, not product code."""
from __future__ import annotations

import hashlib

import numpy as np

from . import instances as I

JITTER = 0.01  # experiment.hpp:47 init_jitter


def sha(*arrays) -> str:
    """SHA-256 over dtype, shape and bytes of each array (None allowed)."""
    h = hashlib.sha256()
    for a in arrays:
        if a is None:
            h.update(b"none")
        else:
            a = np.ascontiguousarray(a)
            h.update(str(a.dtype).encode() + str(a.shape).encode())
            h.update(a.tobytes())
    return h.hexdigest()


def jitter_seed(base: int) -> int:
    return I.mix_seed(base, 7)


def c1(jit=False):
    inst = I.config1(seed=0)
    init = I.jittered_product(inst.mu, inst.nu, JITTER, jitter_seed(1)) if jit else None
    return inst, init


def c2(jit=False):
    return I.config2(seed=0), None


def c3(jit=False):
    inst = I.config3(seed=0)
    init = I.jittered_product(inst.mu, inst.nu, JITTER, jitter_seed(3)) if jit else None
    return inst, init


def c4(n=20000, jit=False, algorithm="bapg"):
    inst = I.config4(seed=0, n=n, algorithm=algorithm)
    init = I.jittered_product(inst.mu, inst.nu, JITTER, jitter_seed(4)) if jit else None
    return inst, init


# name -> (builder, solver-config overrides, full coupling stored)
CASES = {
    "c1": (lambda: c1(), {}, True),
    "c1_jit": (lambda: c1(True), {}, True),
    "c3": (lambda: c3(), {}, True),
    "c3_jit": (lambda: c3(True), {}, True),
    "c2": (lambda: c2(), {}, True),
    "c4_ba4000": (lambda: c4(4000), {}, True),
    "c4_ba4000_jit": (lambda: c4(4000, True), {}, True),
    "c4_hbpg_ba4000": (lambda: c4(4000, algorithm="hbpg"), {}, True),
    # hBPG switched by budget before the reference's eBPG phase reaches its
    # exact fp64 fixed point (iteration 9 at n = 4000).
    "c4_hbpg_ba4000_sw8": (lambda: c4(4000, algorithm="hbpg"), {"switch_iters": 8}, True),
    "c4_n20000_it3": (lambda: c4(20000), {"max_iters": 3}, False),
}
