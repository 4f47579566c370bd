"""Numpy model of the BAPG iteration (solvers.cpp:164-177, plain domain,
fp64) with one injected precision effect, compared per record against a
reference fingerprint (tests/golden/fp_<case>.npz).  The evidence behind
DESIGN.md §4a: which arithmetic of the device path the full-size configs
can tolerate.

    python tools/precision_sim.py c1 MODE [ITERS]

MODE combines (underscore-separated):
  st32          iterates rounded to fp32 after every half-step
  g32           the chain output G rounded to fp32
  opNN          both chain GEMM operands rounded to NN significant bits (22: f16x2)
  biasX         G scaled by (1 − X): a systematic accumulation bias
  noiseX        G scaled by (1 + X·N(0,1)) per entry: random chain error
  dNN           D_X, D_Y rounded once to NN significant bits (a fixed model error)
(the fp32-arithmetic variants of the projections were modelled separately
in the round-2 study).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from harness import cases as HC  # noqa: E402


def main():
    name, mode = sys.argv[1], sys.argv[2]
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else None
    z = np.load(os.path.join(ROOT, "tests", "golden", f"fp_{name}.npz"))
    inst, init = HC.CASES[name][0]()
    iters = iters or len(z["trace"])
    dx, dy, mu, nu, rho = inst.dx, inst.dy, inst.mu, inst.nu, inst.solver["rho"]
    f32 = lambda x: x.astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(0)
    parts = mode.split("_")

    def val(prefix):
        for p in parts:
            if p.startswith(prefix) and p != prefix:
                return float(p[len(prefix):])
        return None

    bits = val("op")
    dbits = val("d")
    if dbits:
        m_, e_ = np.frexp(dx)
        dx = np.ldexp(np.round(m_ * 2.0 ** dbits) / 2.0 ** dbits, e_)
        m_, e_ = np.frexp(dy)
        dy = np.ldexp(np.round(m_ * 2.0 ** dbits) / 2.0 ** dbits, e_)

    def rbits(x):
        m, e = np.frexp(x)
        return np.ldexp(np.round(m * 2.0 ** bits) / 2.0 ** bits, e)

    def chain(x):
        if bits:
            return dx @ rbits(rbits(x) @ dy)
        return dx @ x @ dy

    def g_of(x):
        g = chain(x)
        if val("bias"):
            g = g * (1 - val("bias"))
        if val("noise"):
            g = g * (1 + val("noise") * rng.standard_normal(g.shape))
        if "g32" in parts:
            g = f32(g)
        return g

    store = f32 if "st32" in parts else (lambda x: x)
    pi = init if init is not None else np.outer(mu, nu)
    w = store(pi / pi.sum(axis=0, keepdims=True) * nu[None, :])
    ref = z["trace"][:, 1]
    marks = {1, 10, 100, 500, 1000, 1500, 2000, iters}
    for it in range(1, iters + 1):
        e = g_of(w) / rho
        t = w * np.exp(e - e.max(axis=1, keepdims=True))
        pi = store(t / t.sum(axis=1, keepdims=True) * mu[:, None])
        e = g_of(pi) / rho
        t = pi * np.exp(e - e.max(axis=0, keepdims=True))
        w = store(t / t.sum(axis=0, keepdims=True) * nu[None, :])
        if it in marks:
            a = 0.5 * (pi + w)
            obj = -np.sum((dx @ a @ dy) * a)
            msg = f"{name} {mode} {it}: objective rel err {abs(obj - ref[it - 1]) / abs(ref[it - 1]):.2e}"
            if it == iters and "q" in z:
                sc = float(z["scale"])
                msg += f", coupling err {np.abs(a - z['q'] * sc / 65535).max() / sc:.2e}"
            print(msg, flush=True)


if __name__ == "__main__":
    main()
