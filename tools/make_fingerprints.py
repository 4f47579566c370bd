"""Reference fingerprints of the BASELINE.json configs at full size.

TEST INFRASTRUCTURE.  Runs the REFERENCE's own solver code (oracle/_ref:
proj/src/{types,projections,solvers,diagnostics,tasks}.cpp compiled
unmodified against eigen_lite, fp64 GEMM in numpy's OpenBLAS) on the seeded
instances that bench.py and the GPU tests regenerate, and stores compact
fingerprints under tests/golden/fp_*.npz:

* the trace (iter, objective, infeasibility, split gap, rel_change, phase),
  iterations / converged;
* the final coupling quantised to uint16 against its max (resolution
  7.6e-6 of scale, against the 1e-4 parity bound), or — for n = 20000 —
  16 full rows and a 256 × 256 block in fp64;
* per row the 4 largest entries (fp64 value and index, ties by lowest index
  as hard_assignment, tasks.cpp:190-200) and the row / column sums;
* a SHA-256 of the inputs (edge lists / dense D, marginals, initial
  coupling), so a test knows it regenerated the same instance.

Run here (the container that has /root/reference):
    python tools/make_fingerprints.py [case ...]
Existing files are kept unless --force.  Costs on this 8-core host: c1 / c2
/ c3 / c5 minutes each, BA n=4000 x 200 about half an hour, c4 n=20000 x 3
iterations about 20 minutes and 35 GB of RAM.
"""
import hashlib
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from harness import cases as C  # noqa: E402
from harness import instances as I  # noqa: E402
from paper_2205_08115_b200 import abi  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
sha = C.sha


def top4(pi: np.ndarray):
    """Per row the 4 largest entries, stable (lowest index first on ties)."""
    order = np.argsort(-pi, axis=1, kind="stable")[:, :4]
    return order.astype(np.int32), np.take_along_axis(pi, order, axis=1)


def quantise(pi: np.ndarray):
    scale = float(np.abs(pi).max())
    q = np.rint(np.abs(pi) / scale * 65535.0).astype(np.uint16)
    return q, scale


def trace_array(trace):
    return np.array([[t["iter"], t["objective"], t["marginal_infeasibility"], t["split_gap"],
                      t["rel_change"], t["phase"]] for t in trace], dtype=np.float64)


def cfg_vector(cfg):
    return np.array([getattr(cfg, f) for f, _ in abi.Config._fields_], dtype=np.float64)


def solver_config(inst, **over):
    kw = dict(inst.solver)
    kw.update(over)
    kw["algorithm"] = abi.ALGORITHMS[kw["algorithm"]]
    kw["quiet"] = 1
    return abi.default_config(**kw)


def run_case(ref, name, inst, init, cfg, full=True):
    t0 = time.time()
    r = ref.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu, initial=init)
    assert r.code == 0, r.message
    secs = time.time() - t0
    final = np.asarray(r.final)
    idx, val = top4(final)
    out = dict(trace=trace_array(r.trace), config=cfg_vector(cfg), iterations=r.iterations_used,
               converged=r.converged, top_idx=idx, top_val=val, rowsum=final.sum(axis=1),
               colsum=final.sum(axis=0), input_sha=sha(inst.dx, inst.dy, inst.mu, inst.nu, init),
               seconds=secs, n=inst.n, m=inst.m)
    if full:
        q, scale = quantise(final)
        out.update(q=q, scale=scale)
    else:
        rows = np.linspace(0, inst.n - 1, 16).astype(np.int64)
        out.update(rows=rows, row_vals=final[rows, :].copy(), block=final[:256, :256].copy(),
                   scale=float(np.abs(final).max()),
                   dev_scale=float(np.abs(final - np.outer(inst.mu, inst.nu)).max()))
    path = os.path.join(OUT, f"fp_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {r.iterations_used} it in {secs:.1f}s, objective {r.trace[-1]['objective']:.12e}, "
          f"{os.path.getsize(path) / 1e6:.2f} MB", flush=True)


def c5_case(ref, name, count=256, full_count=32):
    objs, tops_i, tops_v, rows, cols, qs, scales, shas, its = [], [], [], [], [], [], [], [], []
    t0 = time.time()
    for k in range(count):
        inst = I.config5_problem(k)
        cfg = solver_config(inst)
        r = ref.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu)
        assert r.code == 0, r.message
        final = np.asarray(r.final)
        i4, v4 = top4(final)
        objs.append([t["objective"] for t in r.trace])
        tops_i.append(i4)
        tops_v.append(v4)
        rows.append(final.sum(axis=1))
        cols.append(final.sum(axis=0))
        shas.append(sha(inst.dx, inst.dy, inst.mu, inst.nu, None))
        its.append(r.iterations_used)
        if k < full_count:
            q, s = quantise(final)
            qs.append(q)
            scales.append(s)
    path = os.path.join(OUT, f"fp_{name}.npz")
    # Problems may stop early (rel_change exactly 0 <= rel_tol): pad with NaN.
    width = max(len(o) for o in objs)
    obj = np.full((count, width), np.nan)
    for k, o in enumerate(objs):
        obj[k, : len(o)] = o
    np.savez_compressed(path, objective=obj, top_idx=np.array(tops_i),
                        top_val=np.array(tops_v), rowsum=np.array(rows), colsum=np.array(cols),
                        q=np.array(qs), scale=np.array(scales), input_sha=np.array(shas),
                        iterations=np.array(its), config=cfg_vector(cfg), count=count,
                        seconds=time.time() - t0)
    print(f"{name}: {count} problems in {time.time() - t0:.1f}s, "
          f"{os.path.getsize(path) / 1e6:.2f} MB", flush=True)


def case(name):
    make, over, full = C.CASES[name]

    def go(ref):
        inst, init = make()
        run_case(ref, name, inst, init, solver_config(inst, **over), full=full)
    return go


CASES = {name: case(name) for name in C.CASES}
CASES["c5"] = lambda ref: c5_case(ref, "c5")


def main():
    from oracle.bindings import Oracle
    force = "--force" in sys.argv
    names = [a for a in sys.argv[1:] if not a.startswith("--")] or list(CASES)
    ref = Oracle("reference")
    os.makedirs(OUT, exist_ok=True)
    for name in names:
        if not force and os.path.exists(os.path.join(OUT, f"fp_{name}.npz")):
            print(f"{name}: exists, skipped")
            continue
        CASES[name](ref)


if __name__ == "__main__":
    main()
