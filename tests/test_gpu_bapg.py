"""BAPG parity: the B200 path through the C-ABI against the CPU oracle
(oracle/gw_oracle.c, pinned to the reference TUs) on identical seeded inputs.

Tolerances (BASELINE.json north_star): final coupling within 1e-4 max-abs
relative to its scale, GW objective within 1e-5 relative, identical argmax
matching on rows whose oracle top-2 margin exceeds the fp32 error bound.
"""
import numpy as np
import pytest

import paper_2205_08115_b200 as gw
from paper_2205_08115_b200 import abi
from harness import instances as I

pytestmark = pytest.mark.gpu

PI_TOL = 1e-4
OBJ_TOL = 1e-5


def run_both(port, inst, precision, **over):
    solver = dict(inst.solver)
    solver.update(over)
    cfg = gw.SolverConfig(precision=precision, quiet=True, **solver)
    rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                   gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)
    ores = port.solve(cfg.to_abi(), inst.dx, inst.dy, inst.mu, inst.nu)
    assert ores.code == 0, ores.message
    return rep, ores


def rel_scale(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def check_argmax(pi, pi_ref, tol):
    ref_idx = np.argmax(pi_ref, axis=1)
    got = gw.hard_assignment(pi)
    srt = np.sort(pi_ref, axis=1)
    margin = (srt[:, -1] - srt[:, -2]) / np.abs(pi_ref).max()
    decided = margin > 4 * tol
    assert np.array_equal(got[decided], ref_idx[decided]), \
        f"{np.sum(got[decided] != ref_idx[decided])} decided rows differ"
    return decided.mean()


@pytest.mark.parametrize("precision", ["auto", "tf32", "3xtf32", "bf16x3", "bf16x2", "f16x2"])
def test_bapg_er_small(gpu, port, precision):
    inst = I.config1(seed=3, n=256)
    rep, o = run_both(port, inst, precision, max_iters=60)
    assert rep.iterations_used == o.iterations_used == 60
    assert rel_scale(rep.final_coupling.entries(), o.final) < PI_TOL
    assert rel_scale(rep.pi_half.entries(), o.pi) < PI_TOL
    assert rel_scale(rep.w_half.entries(), o.w) < PI_TOL
    obj, obj_ref = rep.trace[-1].objective, o.trace[-1]["objective"]
    # 1xTF32 is the opt-in fast mode: it meets the π bound but not the 1e-5
    # objective bound, so it is held to 2e-4 here.
    assert abs(obj - obj_ref) <= (2e-4 if precision == "tf32" else OBJ_TOL) * abs(obj_ref)
    check_argmax(rep.final_coupling.entries(), o.final, PI_TOL)
    for r, q in zip(rep.trace, o.trace):
        assert r.iter == q["iter"]
        assert abs(r.objective - q["objective"]) <= 2e-4 * abs(q["objective"])
        assert abs(r.rel_change - q["rel_change"]) <= 1e-3 * q["rel_change"] + 1e-7
        assert abs(r.split_gap - q["split_gap"]) <= 1e-3 * q["split_gap"] + 1e-9


@pytest.mark.parametrize("precision", ["auto", "3xtf32", "bf16x3", "f16x2", "f16x3", "tf32"])
def test_bapg_gmm_small(gpu, port, precision):
    # Euclidean distances are not exact in bf16 / fp16: bf16x3 and f16x2 must
    # fall back to 3xTF32; AUTO and f16x3 split both operands.  All of them
    # run on the centred structure matrices, 1xTF32 included
    # (the opt-in fast mode: 11-bit operands, held to looser bounds).
    inst = I.config2(seed=1, n=320, m=256)
    rep, o = run_both(port, inst, precision, max_iters=40)
    tf32 = precision == "tf32"
    assert rel_scale(rep.final_coupling.entries(), o.final) < (2e-3 if tf32 else PI_TOL)
    obj, obj_ref = rep.trace[-1].objective, o.trace[-1]["objective"]
    assert abs(obj - obj_ref) <= (2e-4 if tf32 else OBJ_TOL) * abs(obj_ref)


@pytest.mark.parametrize("precision", ["auto", "3xtf32"])
def test_bapg_weighted_ragged_nonuniform(gpu, port, precision):
    # The centred chain on sizes that are not multiples of the
    # tiles, with non-uniform marginals: the rank-1 biases use rowsum(w) from
    # the column write pass and rowsum(π) = μ, and GEMM2's bias comes from
    # GEMM1's row partials over ragged tiles.
    rng = np.random.default_rng(11)
    base = I.config2(seed=5, n=333, m=201)
    mu = rng.uniform(0.2, 1.8, base.n)
    nu = rng.uniform(0.2, 1.8, base.m)
    inst = I.Instance("gmm_ragged", base.dx, base.dy, mu / mu.sum(), nu / nu.sum(), dict(base.solver))
    rep, o = run_both(port, inst, precision, max_iters=50)
    assert rel_scale(rep.final_coupling.entries(), o.final) < PI_TOL
    assert rel_scale(rep.pi_half.entries(), o.pi) < PI_TOL
    obj, obj_ref = rep.trace[-1].objective, o.trace[-1]["objective"]
    assert abs(obj - obj_ref) <= OBJ_TOL * abs(obj_ref)
    for r, q in zip(rep.trace, o.trace):
        assert abs(r.objective - q["objective"]) <= 2e-4 * abs(q["objective"])
        assert abs(r.marginal_infeasibility - q["marginal_infeasibility"]) <= \
            1e-3 * q["marginal_infeasibility"] + 1e-9


def test_bapg_marginal_invariants(gpu):
    inst = I.config1(seed=5, n=160)
    rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                   gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu),
                   gw.SolverConfig(max_iters=20, rel_tol=1e-30))
    pi, w = rep.pi_half.entries(), rep.w_half.entries()
    # SPEC.md:329 / types.cpp:137-152: each half satisfies its own marginal.
    assert np.abs(pi.sum(axis=1) - inst.mu).max() <= 1e-10
    assert np.abs(w.sum(axis=0) - inst.nu).max() <= 1e-10
    assert abs(rep.final_coupling.entries().sum() - 1.0) <= 1e-9


@pytest.mark.parametrize("precision", ["auto", "fp32"])
def test_bapg_skinny_partition(gpu, port, precision):
    # c3 shape class (m ≤ 32): AUTO runs the skinny bf16x3 chain (FP32-pipe
    # GEMM1 → tensor-core GEMM2 with split-K, csrc/skinny_tc.cu) for a 0/1
    # D_X; "fp32" forces the FP32-pipe chain (csrc/skinny.cu).
    inst = I.config3(seed=2, n=700, k=20)
    rep, o = run_both(port, inst, precision, max_iters=50)
    assert rep.iterations_used == o.iterations_used
    assert rel_scale(rep.final_coupling.entries(), o.final) < PI_TOL
    assert rel_scale(rep.pi_half.entries(), o.pi) < PI_TOL
    obj, obj_ref = rep.trace[-1].objective, o.trace[-1]["objective"]
    assert abs(obj - obj_ref) <= OBJ_TOL * abs(obj_ref)
    check_argmax(rep.final_coupling.entries(), o.final, PI_TOL)


@pytest.mark.parametrize("precision", ["auto", "fp32"])
def test_bapg_skinny_ragged_k(gpu, port, precision):
    # every N class of the skinny kernels' dispatch (m = 1, 5, 13, 32),
    # ragged n (row tiles and k-blocks with tails)
    for k, n in ((1, 300), (5, 333), (13, 129), (32, 517)):
        inst = I.config3(seed=k, n=n, k=k)
        rep, o = run_both(port, inst, precision, max_iters=20)
        assert rel_scale(rep.final_coupling.entries(), o.final) < PI_TOL, k
        obj, obj_ref = rep.trace[-1].objective, o.trace[-1]["objective"]
        assert abs(obj - obj_ref) <= OBJ_TOL * abs(obj_ref), k


_SKINNY_SCRIPT = """
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2205_08115_b200 as gw
from harness import instances as I
out = {{}}
for k, n in ((20, 700), (32, 517), (5, 333), (20, 4000)):
    inst = I.config3(seed=k, n=n, k=k)
    solver = dict(inst.solver); solver.update(max_iters=12)
    cfg = gw.SolverConfig(precision="auto", quiet=True, **solver)
    rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                   gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)
    out[f"pi_{{k}}_{{n}}"] = rep.pi_half.entries()
    out[f"w_{{k}}_{{n}}"] = rep.w_half.entries()
    out[f"obj_{{k}}_{{n}}"] = np.array([r.objective for r in rep.trace])
np.savez(sys.argv[1], **out)
"""


def test_bapg_skinny_fused_half_step_is_bitwise_the_unfused_chain(gpu, tmp_path):
    # csrc/skinny_tc.cu kEpi = 1 (GEMM2 + row update + next GEMM1 in one
    # launch) against one launch per stage (GWB_SKINNY_UNFUSED=1, read once per
    # process): same arithmetic, so iterates and trace are bit-identical —
    # cluster sizes 4 (n = 4000), 5 and 6, ragged last row tiles, m = 5/20/32.
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "skinny_ab.py"
    script.write_text(_SKINNY_SCRIPT.format(root=root))
    res = {}
    for tag, val in (("fused", None), ("unfused", "1")):
        env = dict(os.environ)
        env.pop("GWB_SKINNY_UNFUSED", None)
        if val:
            env["GWB_SKINNY_UNFUSED"] = val
        out = tmp_path / f"{tag}.npz"
        subprocess.run([sys.executable, str(script), str(out)], check=True, env=env, timeout=600)
        res[tag] = np.load(out)
    for key in res["fused"].files:
        assert np.array_equal(res["fused"][key], res["unfused"][key]), key


_COL_SCRIPT = """
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2205_08115_b200 as gw
from harness import instances as I
out = {{}}
for name, inst in (("c1_256", I.config1(n=256)), ("c1_1000", I.config1()), ("c3_700", I.config3(seed=2, n=700, k=20))):
    solver = dict(inst.solver); solver.update(max_iters=10)
    cfg = gw.SolverConfig(precision="auto", quiet=True, **solver)
    rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                   gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)
    out["w_" + name] = rep.w_half.entries()
    out["obj_" + name] = np.array([r.objective for r in rep.trace])
np.savez(sys.argv[1], **out)
"""


def test_bapg_short_column_partials_agree_with_the_online_pass(gpu, tmp_path):
    # csrc/kernels.cu col_partial_short_kernel (max first, independent
    # exponentials; single-wave grids) against the online (max, Σ) pass
    # (GWB_COL_ONLINE=1): the same fp64 column normalisers up to summation
    # order, so 10 iterations agree to ~1e-12 of scale.
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "col_ab.py"
    script.write_text(_COL_SCRIPT.format(root=root))
    res = {}
    for tag, val in (("short", None), ("online", "1")):
        env = dict(os.environ)
        env.pop("GWB_COL_ONLINE", None)
        if val:
            env["GWB_COL_ONLINE"] = val
        out = tmp_path / f"{tag}.npz"
        subprocess.run([sys.executable, str(script), str(out)], check=True, env=env, timeout=600)
        res[tag] = np.load(out)
    for key in res["short"].files:
        a, b = res["short"][key], res["online"][key]
        assert np.abs(a - b).max() <= 1e-10 * np.abs(b).max(), (key, np.abs(a - b).max() / np.abs(b).max())


def test_bapg_skinny_full_c3(gpu, port):
    # BASELINE c3 at full size (n = 4000, K = 20): 32 row tiles × 4 K splits.
    inst = I.config3()
    rep, o = run_both(port, inst, "auto", max_iters=30)
    assert rel_scale(rep.final_coupling.entries(), o.final) < PI_TOL
    obj, obj_ref = rep.trace[-1].objective, o.trace[-1]["objective"]
    assert abs(obj - obj_ref) <= OBJ_TOL * abs(obj_ref)
    check_argmax(rep.final_coupling.entries(), o.final, PI_TOL)


def test_bapg_skinny_weighted_d_takes_fp32_pipes(gpu, port):
    # m ≤ 32 with a non-bf16-exact D_X (Euclidean): AUTO keeps the FP32 chain.
    g = I.config2(seed=5, n=300, m=24)
    rep, o = run_both(port, g, "auto", max_iters=20)
    assert rel_scale(rep.final_coupling.entries(), o.final) < PI_TOL
    obj, obj_ref = rep.trace[-1].objective, o.trace[-1]["objective"]
    assert abs(obj - obj_ref) <= OBJ_TOL * abs(obj_ref)


def test_concurrent_solves_are_reentrant_and_deterministic(gpu):
    # SURVEY §8(b) threading contract: concurrent solve() calls on distinct
    # inputs (the experiment worker pool) are safe and deterministic — each
    # call owns its stream and workspace.
    import threading
    insts = [I.config1(seed=s, n=200 + 40 * s) for s in range(4)]

    def one(inst):
        cfg = gw.SolverConfig(rho=0.1, max_iters=30, rel_tol=1e-30, quiet=True)
        return gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                        gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)

    sequential = [one(x).final_coupling.entries() for x in insts]
    out = [None] * len(insts)
    errs = []

    def worker(k):
        try:
            out[k] = one(insts[k]).final_coupling.entries()
        except Exception as e:  # surfaced below
            errs.append(e)

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(len(insts))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errs, errs
    for a, b in zip(out, sequential):
        assert np.array_equal(a, b)


# f16x2 (AUTO for fp16-exact structure matrices on the single-GPU engine):
# D in fp16 × two fp16 planes of the power-of-two-scaled iterate.  The cases
# below stress the scaling: hub-heavy BA degrees, non-uniform
# and ragged marginals, integer weights > 1, and a coupling driven far from
# uniform (small ρ, many iterations) so its entries span many binades.
def _f16_case(port, inst, **over):
    rep, o = run_both(port, inst, "auto", **over)
    assert rep.iterations_used == o.iterations_used
    assert rel_scale(rep.final_coupling.entries(), o.final) < PI_TOL
    assert rel_scale(rep.pi_half.entries(), o.pi) < PI_TOL
    assert rel_scale(rep.w_half.entries(), o.w) < PI_TOL
    for r, q in zip(rep.trace, o.trace):
        assert abs(r.objective - q["objective"]) <= OBJ_TOL * abs(q["objective"])
    check_argmax(rep.final_coupling.entries(), o.final, PI_TOL)
    return rep, o


def _session_precision(inst, precision):
    import ctypes as C
    import torch
    lib = abi.load()
    cfg = gw.SolverConfig(precision=precision, quiet=True, max_iters=4).to_abi()
    st = abi.Status()
    sess = C.c_void_p()
    n, m = inst.dx.shape[0], inst.dy.shape[0]
    lib.gwb_session_create(C.byref(cfg), n, m, 0, C.byref(sess), C.byref(st))
    abi.raise_for(st)
    dev = dict(device="cuda", dtype=torch.float32)
    dx, dy = torch.tensor(inst.dx, **dev), torch.tensor(inst.dy, **dev)
    mu, nu = torch.tensor(inst.mu, **dev), torch.tensor(inst.nu, **dev)
    lib.gwb_session_load_device(sess, dx.data_ptr(), n, dy.data_ptr(), m, mu.data_ptr(),
                                nu.data_ptr(), None, C.byref(st))
    abi.raise_for(st)
    rprec, flops = C.c_int32(0), C.c_double(0)
    lib.gwb_session_info(sess, C.byref(rprec), C.byref(flops), C.byref(st))
    lib.gwb_session_destroy(sess)
    return rprec.value


def test_f16x2_is_auto_for_graphs(gpu):
    # 0/1 graphs resolve AUTO to f16x2; Euclidean D (not fp16-exact) to f16x3
    # (both operands split); an explicit f16x2 request on such D falls back
    # f16x2 -> bf16x3 -> 3xTF32.
    assert _session_precision(I.config1(seed=3, n=256), "auto") == abi.PREC_F16X2
    gmm = I.config2(seed=1, n=320, m=256)
    assert _session_precision(gmm, "auto") == abi.PREC_F16X3
    assert _session_precision(gmm, "f16x2") == abi.PREC_3XTF32


def test_f16x2_ba_hubs(gpu, port):
    inst = I.config4(n=1024)
    _f16_case(port, inst, max_iters=200)


def test_f16x2_nonuniform_ragged(gpu, port):
    rng = np.random.default_rng(11)
    base = I.config1(seed=4, n=300)
    n, m = 300, 260
    dx = base.dx
    dy = base.dy[:m, :m].copy()
    mu = rng.uniform(0.05, 3.0, n)
    mu /= mu.sum()
    nu = rng.uniform(0.05, 3.0, m) ** 3
    nu /= nu.sum()
    inst = I.Instance(name="ragged", dx=dx, dy=dy, mu=mu, nu=nu, solver=dict(base.solver))
    _f16_case(port, inst, max_iters=120)


def test_f16x2_integer_weights(gpu, port):
    # Hop-count-like integer weights up to 40: exact in fp16, Vᵀ row bounds
    # scale with the weighted degrees.
    rng = np.random.default_rng(5)
    base = I.config1(seed=6, n=288)
    w = rng.integers(1, 41, size=base.dx.shape)
    w = np.triu(w, 1) + np.triu(w, 1).T
    dx = base.dx * w
    dy = base.dy * w
    inst = I.Instance(name="weighted", dx=dx, dy=dy, mu=base.mu, nu=base.nu,
                      solver=dict(base.solver, rho=5.0))
    _f16_case(port, inst, max_iters=80)


@pytest.mark.parametrize("precision", ["auto", "bf16x3"])
def test_concentrated_coupling(gpu, port, precision):
    # ρ = 0.05, 300 iterations: the coupling has found the permutation (max
    # entry 1/n) and its entries span > 100 binades (some below fp32's
    # normal range), far outside the scale the f16x2 bounds are tight for.
    inst = I.config1(seed=8, n=256)
    rep, o = run_both(port, inst, precision, max_iters=300, rho=0.05)
    fin = o.final[o.final > 1e-300]
    assert np.log2(fin.max() / fin.min()) > 100
    assert rel_scale(rep.final_coupling.entries(), o.final) < PI_TOL
    assert rel_scale(rep.pi_half.entries(), o.pi) < PI_TOL
    for r, q in zip(rep.trace, o.trace):
        assert abs(r.objective - q["objective"]) <= OBJ_TOL * abs(q["objective"])
    check_argmax(rep.final_coupling.entries(), o.final, PI_TOL)


def test_f16x2_auto_large_nonuniform(gpu, port):
    """The headline chain (f16x2, AUTO for 0/1 graphs) at c4-scale K with
    non-uniform marginals: the power-of-two iterate scale (from max μ, ν),
    the per-row Vᵀ scales and the fp16 Vᵀ planes all in play,
    against the oracle (fp64) over the first iterations."""
    n = 8192
    inst = I.alignment_instance(I.barabasi_albert(n, 5, 77), n, 0.02, 77, "ba8192", {})
    rng = np.random.default_rng(5)
    mu = rng.uniform(0.2, 1.8, n)
    nu = rng.uniform(0.2, 1.8, n)
    mu, nu = mu / mu.sum(), nu / nu.sum()
    cfg = gw.SolverConfig(rho=0.1, max_iters=3, rel_tol=1e-30, quiet=True)
    assert _session_precision(inst, "auto") == abi.PREC_F16X2
    rep = gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                   gw.ProbabilityVector(mu), gw.ProbabilityVector(nu), cfg)
    o = port.solve(cfg.to_abi(), inst.dx, inst.dy, mu, nu)
    assert o.code == 0
    np.testing.assert_allclose([r.objective for r in rep.trace], [t["objective"] for t in o.trace],
                               rtol=1e-6)
    pi, ref = rep.final_coupling.entries(), o.final
    assert np.abs(pi - ref).max() <= 1e-6 * np.abs(ref).max()
    # the deviation from the start is what 3 iterations produce: hold it too
    dev, dev_ref = pi - np.outer(mu, nu), ref - np.outer(mu, nu)
    assert np.abs(dev - dev_ref).max() <= 1e-3 * np.abs(dev_ref).max()
