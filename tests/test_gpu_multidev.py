"""In-library multi-device execution behind the drop-in boundary (gwb_set_devices
/ GWB_DEVICES): a C caller gets several GPUs with no torch.

* gwb_solve with more than one device row-shards one BAPG problem over them
  (shard.cu: the sharded engines + NCCL's single-process communicator).  On a
  one-GPU box the device is listed twice, which runs the same schedule with
  emulated collectives — the orchestration, row layout and output assembly
  are exercised; NCCL itself is covered by the torch.distributed path.
* gwb_bapg_solve_batched splits the problems into contiguous ranges, one host
  thread per device, no communication.
"""
import ctypes as C

import numpy as np
import pytest

import paper_2205_08115_b200 as gw
from harness import instances as I
from paper_2205_08115_b200 import abi

pytestmark = pytest.mark.gpu


def set_devices(ids):
    st = abi.Status()
    arr = (C.c_int32 * len(ids))(*ids)
    rc = abi.load().gwb_set_devices(len(ids), arr, C.byref(st))
    assert rc == 0, st.message


@pytest.fixture
def two_ranks(gpu):
    set_devices([0, 0])
    yield
    set_devices([0])


def solve(inst, **kw):
    cfg = gw.SolverConfig(quiet=True, **{**inst.solver, **kw})
    return cfg, gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                         gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)


@pytest.mark.parametrize("case", ["er", "gmm"])
def test_sharded_solve_matches_oracle(two_ranks, port, case):
    inst = I.config1(seed=31, n=300) if case == "er" else I.config2(seed=32, n=260, m=200)
    cfg, rep = solve(inst, max_iters=50, rel_tol=1e-30)
    o = port.solve(cfg.to_abi(), inst.dx, inst.dy, inst.mu, inst.nu)
    assert o.code == 0
    assert rep.iterations_used == o.iterations_used == 50
    scale = np.abs(o.final).max()
    assert np.abs(rep.final_coupling.entries() - o.final).max() <= 1e-4 * scale
    assert np.abs(rep.pi_half.entries() - o.pi).max() <= 1e-4 * np.abs(o.pi).max()
    obj = [r.objective for r in rep.trace]
    np.testing.assert_allclose(obj, [t["objective"] for t in o.trace], rtol=1e-5)
    # π rows sum to μ exactly in fp64 (the shard iterates are fp64)
    np.testing.assert_allclose(rep.pi_half.entries().sum(axis=1), inst.mu, rtol=1e-12)


def test_sharded_stop_rule_and_ragged_rows(two_ranks, port):
    # n not a multiple of the 64-row shard granularity; a reachable tolerance.
    inst = I.alignment_instance(I.barabasi_albert(150, 3, 5), 150, 0.05, 5, "ba150", {})
    cfg, rep = solve(inst, rho=0.1, max_iters=400, rel_tol=1e-6)
    o = port.solve(cfg.to_abi(), inst.dx, inst.dy, inst.mu, inst.nu)
    assert o.code == 0 and o.converged and rep.converged
    assert abs(rep.iterations_used - o.iterations_used) <= 1


def test_sharded_overflow_error(two_ranks, port):
    inst = I.config1(seed=2, n=130)
    cfg = gw.SolverConfig(quiet=True, rho=1e-6, max_iters=10)
    o = port.solve(cfg.to_abi(), inst.dx, inst.dy, inst.mu, inst.nu)
    with pytest.raises(gw.NumericalInstabilityError) as e:
        gw.solve(gw.DistanceMatrix.trusted(inst.dx), gw.DistanceMatrix.trusted(inst.dy),
                 gw.ProbabilityVector(inst.mu), gw.ProbabilityVector(inst.nu), cfg)
    assert str(e.value) == o.message


def test_batched_split_matches_single_device(gpu):
    probs = [I.config5_problem(k) for k in range(7)]
    cfg = gw.SolverConfig(quiet=True, **probs[0].solver)
    args = ([gw.DistanceMatrix.trusted(p.dx) for p in probs],
            [gw.DistanceMatrix.trusted(p.dy) for p in probs],
            [gw.ProbabilityVector(p.mu) for p in probs],
            [gw.ProbabilityVector(p.nu) for p in probs])
    one = gw.bapg_solve_batched(*args, cfg)
    set_devices([0, 0, 0])
    try:
        three = gw.bapg_solve_batched(*args, cfg)
    finally:
        set_devices([0])
    for a, b in zip(one, three):
        assert a.iterations_used == b.iterations_used
        np.testing.assert_array_equal(a.final_coupling.entries(), b.final_coupling.entries())
        assert [r.objective for r in a.trace] == [r.objective for r in b.trace]
