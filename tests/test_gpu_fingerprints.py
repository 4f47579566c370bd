"""Full-size parity: the B200 path (AUTO precision, the bench's chains)
against fingerprints of the REFERENCE's own solver on the BASELINE.json
configs at their stated sizes and iteration counts.

The fingerprints (tests/golden/fp_*.npz) were made by tools/make_fingerprints.py
with oracle/_ref (the reference's solvers.cpp / projections.cpp / types.cpp
compiled unmodified, fp64 GEMM in OpenBLAS).  Here the seeded inputs are
regenerated (harness/cases.py; the input SHA-256 must match), solved
through the C-ABI (gwb_solve via the gw:: mirror, gwb_bapg_solve_batched for
c5) and compared:

* every trace objective within 1e-5 relative (final record: relative to
  itself; earlier records: relative to the largest |objective|);
* the final coupling within 1e-4 max-abs relative to its scale (the stored
  copy is quantised to 7.6e-6 of scale, which is charged to the bound);
* row / column sums of the final coupling;
* argmax parity (tests/parity.py) with a minimum decided-row fraction;
* iterations used / converged.
"""
import os

import numpy as np
import pytest

import paper_2205_08115_b200 as gw
from harness import cases as C
from harness import instances as I
from tests.parity import OBJ_TOL, PI_TOL, QUANT, argmax_check, dequantise

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(__file__), "golden")

# Minimum decided fraction per case.  c3 from the product start is an exact
# symmetric fixed point of the reference (every row a 20-way exact tie,
# checked through the tied-set rule); after 3 iterations at n = 20000 the
# coupling has barely left the product start.
MIN_DECIDED = {"c1": 0.9, "c1_jit": 0.9, "c3": 0.0, "c3_jit": 0.9, "c2": 0.9,
               "c4_ba4000": 0.9, "c4_ba4000_jit": 0.9, "c4_hbpg_ba4000_sw8": 0.8,
               "c4_n20000_it3": 0.0}


def load(name):
    path = os.path.join(HERE, f"fp_{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing fingerprint {path} (tools/make_fingerprints.py)")
    return np.load(path)


def solve_case(name):
    make, over, _ = C.CASES[name]
    inst, init = make()
    solver = dict(inst.solver)
    solver.update(over)
    cfg = gw.SolverConfig(quiet=True, **solver)
    rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                   gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg,
                   gw.SolveOptions(initial=init) if init is not None else None)
    return inst, init, rep


def check_trace(rep, z, label):
    want = z["trace"]
    got = np.array([[r.iter, r.objective, r.phase] for r in rep.trace])
    assert got.shape[0] == want.shape[0], (got.shape, want.shape)
    np.testing.assert_array_equal(got[:, 0], want[:, 0])
    np.testing.assert_array_equal(got[:, 2], want[:, 5])  # hBPG phases
    obj, obj_ref = got[:, 1], want[:, 1]
    scale = np.abs(obj_ref).max()
    err_all = np.abs(obj - obj_ref).max() / scale
    err_final = abs(obj[-1] - obj_ref[-1]) / abs(obj_ref[-1])
    print(f"{label}: objective final rel err {err_final:.2e}, all records {err_all:.2e}")
    assert err_final <= OBJ_TOL
    assert err_all <= OBJ_TOL


@pytest.mark.parametrize("name", ["c1", "c1_jit", "c3", "c3_jit", "c2", "c4_ba4000",
                                  "c4_ba4000_jit", "c4_hbpg_ba4000_sw8"])
def test_fingerprint_full_coupling(gpu, name):
    z = load(name)
    inst, init, rep = solve_case(name)
    assert C.sha(inst.dx, inst.dy, inst.mu, inst.nu, init) == str(z["input_sha"]), \
        "regenerated inputs differ from the fingerprint's"
    assert rep.iterations_used == int(z["iterations"])
    assert rep.converged == bool(z["converged"])
    check_trace(rep, z, name)
    pi = rep.final_coupling.entries()
    scale = float(z["scale"])
    ref = dequantise(z["q"], scale)
    err = np.abs(pi - ref).max() / scale
    print(f"{name}: coupling err {err:.2e} of scale (+{QUANT:.1e} quantisation)")
    assert err + QUANT <= PI_TOL
    np.testing.assert_allclose(pi.sum(axis=1), z["rowsum"], rtol=0, atol=PI_TOL * np.abs(z["rowsum"]).max())
    np.testing.assert_allclose(pi.sum(axis=0), z["colsum"], rtol=0, atol=PI_TOL * np.abs(z["colsum"]).max())
    pick = gw.hard_assignment(pi)
    argmax_check(pick, pi, z["top_idx"], z["top_val"], MIN_DECIDED[name], name,
                 ref_value_at=lambda r, c: ref[r, c], slack=QUANT * scale)


def test_fingerprint_hbpg_ebpg_phase(gpu):
    """c4 hBPG at n = 4000 with switch_iters = 100: the reference's eBPG phase
    ends at iteration 9 on an exact fp64 fixed point (rel_change 3.9e-16,
    7.6e-17, 7.3e-19, 5.3e-20, then exactly 0), an event decided by the last
    bits of its own summation order; the device's eBPG iterate passes through
    an fp32 chain and cannot see changes below 2^-24, so it switches by budget
    (DESIGN.md §5).  What is compared: the eBPG phase itself — every record
    up to the reference's switch (objective 1e-5, coupling converged to the
    same fixed point: rel_change below 1e-6 from iteration 3 on)."""
    z = load("c4_hbpg_ba4000")
    want = z["trace"]
    k_switch = int((want[:, 5] == 1).sum())
    assert k_switch == 9
    inst, init = C.c4(4000, algorithm="hbpg")
    cfg = gw.SolverConfig(quiet=True, **{**inst.solver, "max_iters": k_switch})
    rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                   gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)
    got = np.array([[r.objective, r.rel_change, r.phase] for r in rep.trace])
    assert got.shape[0] == k_switch and (got[:, 2] == 1).all()
    np.testing.assert_allclose(got[:, 0], want[:k_switch, 1], rtol=OBJ_TOL)
    assert abs(got[0, 1] - want[0, 4]) <= 1e-3 * want[0, 4]   # first step: same move
    assert (got[2:, 1] < 1e-6).all()                          # converged like the reference


def test_fingerprint_c4_n20000_first_iterations(gpu):
    """c4 at n = m = 20000: the first 3 iterations against the reference
    (one reference iteration is minutes of fp64 BLAS).  Beyond the 1e-4
    scale bound, the coupling's deviation from the product start — which is
    what 3 iterations produce — is held to 1e-3 of its own scale."""
    name = "c4_n20000_it3"
    z = load(name)
    inst, init, rep = solve_case(name)
    assert C.sha(inst.dx, inst.dy, inst.mu, inst.nu, init) == str(z["input_sha"])
    assert rep.iterations_used == int(z["iterations"]) == 3
    check_trace(rep, z, name)
    pi = rep.final_coupling.entries()
    rows = z["rows"]
    scale = float(z["scale"])
    err_rows = np.abs(pi[rows, :] - z["row_vals"]).max() / scale
    err_block = np.abs(pi[:256, :256] - z["block"]).max() / scale
    prod = np.outer(inst.mu, inst.nu)
    dev_scale = float(z["dev_scale"])
    dev_rows = np.abs((pi[rows, :] - prod[rows, :]) - (z["row_vals"] - prod[rows, :])).max() / dev_scale
    print(f"{name}: rows err {err_rows:.2e}, block err {err_block:.2e} of scale; "
          f"deviation err {dev_rows:.2e} of the deviation scale {dev_scale:.3e}")
    assert err_rows <= PI_TOL and err_block <= PI_TOL
    assert dev_rows <= 1e-3
    np.testing.assert_allclose(pi.sum(axis=1), z["rowsum"], rtol=1e-6)
    np.testing.assert_allclose(pi.sum(axis=0), z["colsum"], rtol=1e-6)
    # Argmax after 3 iterations: most rows are still near-uniform; the
    # tied/near-tie rules apply to all of them, decided rows must match.
    pick = gw.hard_assignment(pi)
    argmax_check(pick, pi, z["top_idx"], z["top_val"], MIN_DECIDED[name], name)


def test_fingerprint_c5_batched(gpu):
    """c5: 256 of the 4096 problems (n = m = 128, 500 iterations) through
    gwb_bapg_solve_batched (the on-chip batched kernel the bench times)
    against the reference solving each problem."""
    z = load("c5")
    count = int(z["count"])
    insts = [I.config5_problem(k) for k in range(count)]
    for k in (0, count // 2, count - 1):
        i = insts[k]
        assert C.sha(i.dx, i.dy, i.mu, i.nu, None) == str(z["input_sha"][k])
    cfg = gw.SolverConfig(quiet=True, **insts[0].solver)
    reps = gw.bapg_solve_batched([gw.DistanceMatrix.trusted(i.dx) for i in insts],
                                 [gw.DistanceMatrix.trusted(i.dy) for i in insts],
                                 [gw.ProbabilityVector(i.mu) for i in insts],
                                 [gw.ProbabilityVector(i.nu) for i in insts], cfg)
    obj_ref = z["objective"]
    worst_obj, worst_pi, decided, rows, same_stop, early = 0.0, 0.0, 0, 0, 0, []
    for k, rep in enumerate(reps):
        # The reference stops where rel_change crosses the pinned 1e-30
        # (iterations 149-350 for most problems, decaying ×0.6 per iteration);
        # the device stops there too, within one iteration.  The batched
        # kernel's iterates are fp32: where the reference keeps creeping at
        # ~1e-20 relative (no crossing within 500), the fp32 iterate turns
        # bitwise stationary and stops earlier; its coupling has converged,
        # so it must still match the reference's final one (checked below).
        ref_it = int(z["iterations"][k])
        if abs(rep.iterations_used - ref_it) <= 1:
            same_stop += 1
        else:
            assert rep.converged and rep.iterations_used < ref_it, (k, rep.iterations_used, ref_it)
            early.append(k)
        obj = np.array([r.objective for r in rep.trace])[: ref_it]
        want = obj_ref[k][: len(obj)]
        worst_obj = max(worst_obj, np.abs(obj - want).max() / np.abs(want).max())
        fin = obj_ref[k][ref_it - 1]
        worst_obj = max(worst_obj, abs(obj[-1] - fin) / abs(fin))
        pi = rep.final_coupling.entries()
        np.testing.assert_allclose(pi.sum(axis=1), z["rowsum"][k], rtol=0, atol=1e-4 / 128)
        ref_at, slack = None, 0.0
        if k < z["q"].shape[0]:  # full couplings stored for the first 32
            scale = float(z["scale"][k])
            ref = dequantise(z["q"][k], scale)
            err = np.abs(pi - ref).max() / scale
            worst_pi = max(worst_pi, err)
            assert err + QUANT <= PI_TOL, (k, err)
            ref_at, slack = (lambda r, c, ref=ref: ref[r, c]), QUANT * scale
        info = argmax_check(gw.hard_assignment(pi), pi, z["top_idx"][k], z["top_val"][k], 0.0,
                            f"c5[{k}]", ref_value_at=ref_at, slack=slack)
        decided += info["decided"]
        rows += info["rows"]
    print(f"c5: {count} problems, worst objective rel err {worst_obj:.2e}, worst coupling err "
          f"{worst_pi:.2e}, decided rows {decided}/{rows}, stop iteration within one in "
          f"{same_stop}/{count}; earlier fp32-stationary stops: {early}")
    assert same_stop >= 0.9 * count
    assert worst_obj <= OBJ_TOL
    assert decided >= 0.9 * rows
