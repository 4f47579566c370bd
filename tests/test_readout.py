"""Post-solve readout: coupling_entropy,
alignment_accuracy and the device-side session readout of run_cell
(experiment.cpp:169-195).  The oracle's two new leaves are pinned to the
reference build first."""
import ctypes as C

import numpy as np
import pytest

import paper_2205_08115_b200 as gw
from paper_2205_08115_b200 import abi
from harness import instances as I


def _coupling(n=37, m=23, seed=0):
    rng = np.random.default_rng(seed)
    p = rng.random((n, m)) ** 3
    p[rng.random((n, m)) < 0.2] = 0.0  # exact zeros: 0 log 0 := 0
    return np.asfortranarray(p / p.sum())


def test_oracle_entropy_matches_reference(port, ref):
    for seed in range(3):
        p = _coupling(seed=seed)
        a, b = port.coupling_entropy(p), ref.coupling_entropy(p)
        assert abs(a - b) <= 1e-13 * abs(b)


def test_alignment_accuracy_matches_reference(port, ref):
    pred = np.array([0, 2, 2, 5, 1], dtype=np.int32)
    gt = np.array([0, 1, 2, 5], dtype=np.int32)
    for o in (port, ref):
        rc, acc, _ = o.alignment_accuracy(pred, gt)
        assert rc == 0 and acc == 75.0
    assert gw.alignment_accuracy(pred, gt) == 75.0
    rc, _, msg = ref.alignment_accuracy(gt[:2], gt)
    assert rc == abi.ERR_DIMENSION
    with pytest.raises(gw.DimensionMismatchError, match=msg):
        gw.alignment_accuracy(gt[:2], gt)
    rc, _, msg = ref.alignment_accuracy(pred, gt[:0])
    assert rc == abi.ERR_INVALID and msg == "empty ground truth"
    with pytest.raises(ValueError, match="empty ground truth"):
        gw.alignment_accuracy(pred, gt[:0])


@pytest.mark.gpu
def test_coupling_entropy_device(gpu, port):
    for seed in range(3):
        p = _coupling(n=300, m=211, seed=seed)
        assert abs(gw.coupling_entropy(p) - port.coupling_entropy(p)) <= 1e-12 * port.coupling_entropy(p)


@pytest.mark.gpu
def test_session_readout_matches_run_cell(gpu, port):
    import torch
    inst = I.config1(seed=11, n=320)
    n = inst.n
    iters = 60
    lib = abi.load()
    ld = (n + 31) // 32 * 32
    t = lambda a: torch.nn.functional.pad(torch.tensor(np.ascontiguousarray(a), dtype=torch.float32),
                                          (0, ld - a.shape[1])).cuda()
    dx, dy = t(inst.dx), t(inst.dy)
    mu = torch.tensor(inst.mu, dtype=torch.float32).cuda()
    cfg = abi.default_config(rho=0.1, max_iters=iters + 4, rel_tol=1e-30)
    st = abi.Status()
    s = C.c_void_p()
    lib.gwb_session_create(C.byref(cfg), n, n, 0, C.byref(s), C.byref(st))
    abi.raise_for(st)
    try:
        lib.gwb_session_load_device(s, dx.data_ptr(), ld, dy.data_ptr(), ld, mu.data_ptr(),
                                    mu.data_ptr(), None, C.byref(st))
        abi.raise_for(st)
        lib.gwb_session_reset(s, None, C.byref(st))
        lib.gwb_session_iterate(s, iters, None, None, C.byref(st))
        abi.raise_for(st)
        gt = np.ascontiguousarray(inst.ground_truth, dtype=np.int32)
        assign = np.zeros(n, dtype=np.int32)
        out = abi.Readout()
        i32 = C.POINTER(C.c_int32)
        lib.gwb_session_readout(s, gt.ctypes.data_as(i32), n, assign.ctypes.data_as(i32),
                                C.byref(out), C.byref(st))
        abi.raise_for(st)
    finally:
        lib.gwb_session_destroy(s)
    ocfg = abi.default_config(rho=0.1, max_iters=iters, rel_tol=1e-30)
    o = port.solve(ocfg, inst.dx, inst.dy, inst.mu, inst.nu)
    plan = o.final
    rc, obj, _ = port.gw_objective(inst.dx, inst.dy, plan)
    assert rc == 0
    assert abs(out.objective - obj) <= 1e-5 * abs(obj)
    assert abs(out.entropy - port.coupling_entropy(plan)) <= 1e-6 * abs(port.coupling_entropy(plan))
    mi = port.marginal_infeasibility(plan, inst.mu, inst.nu)
    assert abs(out.marginal_infeasibility - mi) <= 1e-3 * mi + 1e-9
    sg = port.split_gap(o.pi, o.w)
    assert abs(out.split_gap - sg) <= 1e-3 * sg + 1e-6 * np.linalg.norm(o.pi)
    ref_assign = port.hard_assignment(plan)
    srt = np.sort(plan, axis=1)
    decided = (srt[:, -1] - srt[:, -2]) / np.abs(plan).max() > 4e-4
    assert np.array_equal(assign[decided], ref_assign[decided])
    assert out.has_accuracy == 1
    rc, acc, _ = port.alignment_accuracy(assign, gt)
    assert rc == 0 and out.accuracy == acc
    rc, res, _ = port.luo_tseng_residual(inst.dx, inst.dy, plan, inst.mu, inst.nu)
    assert rc == 0 and abs(out.residual - res) <= 1e-4 * res
