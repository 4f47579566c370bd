"""Multi-rank host logic on CPU: world_size 2 and 3 over gloo.

Each rank runs the CPU mirror of its shard (tests/shard_mirror.py) through
the product's orchestrator (`dist.run_sharded` + `dist.TorchComm`) with real
torch.distributed collectives; the assembled coupling and trace must equal
the single-process oracle.  This pins the sharding plan, the blocked Vᵀ
all-gather layout, the rank-ordered column merge and the agreed stop rule.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2205_08115_b200 import abi
from harness import instances as I
from paper_2205_08115_b200.dist import ShardPlan


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, iters, rel_tol, q, overlap=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2205_08115_b200.dist import TorchComm, run_sharded
    from tests.shard_mirror import CpuShard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inst = I.config1(seed=9, n=n)
    s = CpuShard(inst.dx, inst.dy, inst.mu, inst.nu, 0.1, rank, world, iters, rel_tol)
    s.reset()
    st = run_sharded([s], TorchComm(dist, rank, world), iters, poll_every=4,
                     overlap=overlap)
    used = st["iter"] - 1
    pi, w = s.rows()
    q.put((rank, pi, w, s.trace(used), st))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, n, iters, rel_tol, overlap=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, iters, rel_tol, q, overlap))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda x: x[0])
    pi = np.vstack([o[1] for o in out])
    w = np.vstack([o[2] for o in out])
    return pi, w, out[0][3], [o[4] for o in out]


@pytest.mark.parametrize("world,n,overlap", [(2, 150, False), (3, 130, False), (2, 150, True),
                                             (3, 130, True)])
def test_sharded_bapg_matches_oracle_gloo(port, world, n, overlap):
    # overlap=True: per-source broadcasts + partial GEMM2s (own block first)
    iters = 12
    pi, w, trace, sts = _run(world, n, iters, 1e-30, overlap)
    inst = I.config1(seed=9, n=n)
    o = port.solve(abi.default_config(rho=0.1, max_iters=iters, rel_tol=1e-30), inst.dx, inst.dy,
                   inst.mu, inst.nu)
    assert o.code == 0
    assert all(s["iter"] - 1 == iters for s in sts)
    np.testing.assert_allclose(pi, o.pi, rtol=0, atol=1e-12 * np.abs(o.pi).max())
    np.testing.assert_allclose(w, o.w, rtol=0, atol=1e-12 * np.abs(o.w).max())
    for r, q in zip(trace, o.trace):
        for k in ("objective", "marginal_infeasibility", "split_gap", "rel_change"):
            assert r[k] == pytest.approx(q[k], rel=1e-9, abs=1e-14), k


@pytest.mark.parametrize("overlap", [False, True])
def test_sharded_stop_rule_agreed_gloo(port, overlap):
    # every rank must stop at the oracle's convergence iteration
    n, iters = 64, 1200
    pi, w, trace, sts = _run(2, n, iters, 1e-6, overlap)
    inst = I.config1(seed=9, n=n)
    o = port.solve(abi.default_config(rho=0.1, max_iters=iters, rel_tol=1e-6), inst.dx, inst.dy,
                   inst.mu, inst.nu)
    assert o.converged
    assert all(s["converged"] == 1 and s["iter"] - 1 == o.iterations_used for s in sts)
    np.testing.assert_allclose(pi, o.pi, rtol=0, atol=1e-12)


def test_shard_plan():
    p = ShardPlan(20000, 8)
    assert p.rows_per_shard == 2560 and p.rows_per_shard % 64 == 0
    assert sum(p.rows_valid(r) for r in range(8)) == 20000
    p = ShardPlan(100, 3)
    assert [p.rows_valid(r) for r in range(3)] == [64, 36, 0]


# ---- row-sharded eBPG / BPG / hBPG orchestration (dist.run_bregman_sharded)

def _bworker(rank, world, port, over, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2205_08115_b200.dist import TorchComm, run_bregman_sharded
    from tests.bshard_mirror import CpuBregShard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inst = I.config1(seed=6, n=90)
    cfg = abi.default_config(rel_tol=1e-30, quiet=1, **over)
    s = CpuBregShard(cfg, inst.dx, inst.dy, inst.mu, inst.nu, rank, world)
    out = run_bregman_sharded([s], TorchComm(dist, rank, world),
                              cfg.max_iters)[0]
    q.put((rank, out["final"], [t["objective"] for t in out["trace"]],
           [t["phase"] for t in out["trace"]], out["iterations_used"]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("over", [
    dict(algorithm=abi.HBPG, epsilon_reg=0.1, step=5.0, inner_iters=10, switch_iters=3, max_iters=7),
    dict(algorithm=abi.BPG, step=5.0, inner_iters=10, max_iters=5, perturbation=0.01),
], ids=["hbpg", "bpg"])
def test_sharded_bregman_matches_oracle_gloo(port, world, over):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pno = _free_port()
    procs = [ctx.Process(target=_bworker, args=(r, world, pno, over, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    inst = I.config1(seed=6, n=90)
    cfg = abi.default_config(rel_tol=1e-30, quiet=1, **over)
    o = port.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu)
    assert o.code == 0, o.message
    for _, final, objs, phases, used in res:
        assert used == o.iterations_used
        assert np.abs(final - o.final).max() <= 1e-10 * np.abs(o.final).max()
        np.testing.assert_allclose(objs, [t["objective"] for t in o.trace], rtol=1e-9)
        assert phases == [t["phase"] for t in o.trace]


def _agree_worker(rank, world, port, values, q, request=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2205_08115_b200 import dist as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = np.zeros((4, 8), dtype=np.float32)
    rows[0, 1] = values[rank]  # this rank's rows of D_X
    dy = np.eye(8, dtype=np.float32)
    cfg = D.resolve_precision(abi.default_config(), True)  # pass-through check below
    req = abi.default_config() if request is None else abi.default_config(precision=request)
    assert D.needs_agreement(req)
    out = D._agree_precision(req, rows, dy, dist, 0)
    q.put((rank, out.precision, cfg.precision))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("values,expect", [
    ((1.0, 1.0), abi.PREC_F16X2),               # 0/1 rows everywhere
    ((1.0, 2.0 ** 20), abi.PREC_BF16X3),        # rank 1: exact in bf16, beyond fp16 range
    ((1.0, 1.0 / 3.0), abi.PREC_3XTF32),        # rank 1: exact in neither
])
def test_auto_precision_agreed_across_ranks(values, expect):
    # dist._agree_precision: every rank tests its own rows; the MIN
    # all-reduce of the bf16 / fp16 verdicts makes all ranks pick one chain.
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, 2, port, values, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(o[1] == expect for o in out), out
    assert all(o[2] == abi.PREC_BF16X3 for o in out)  # explicit exact flag, no fp16 verdict


@pytest.mark.parametrize("request_prec,values,expect", [
    (abi.PREC_F16X2, (1.0, 1.0), abi.PREC_F16X2),
    (abi.PREC_F16X2, (1.0, 2.0 ** 20), abi.PREC_BF16X3),   # weighted beyond fp16 on rank 1
    (abi.PREC_F16X2, (0.7, 1.0), abi.PREC_3XTF32),         # rank 0: exact in neither
    (abi.PREC_BF16X3, (1.0, 1.0 / 3.0), abi.PREC_3XTF32),
    (abi.PREC_BF16X2, (1.0, 2.0 ** 20), abi.PREC_BF16X2),  # bf16-exact: kept
])
def test_explicit_split_precision_downgraded_across_ranks(request_prec, values, expect):
    # An explicit f16x2 / bf16x3 / bf16x2 request on a weighted D must not
    # round D silently: every rank agrees on the exactness and
    # falls back as the single-GPU engine does (f16x2 -> bf16x3 -> 3xTF32).
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, 2, port, values, q, request_prec))
             for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(o[1] == expect for o in out), out


def test_resolve_precision_passthrough_for_tf32_chains():
    from paper_2205_08115_b200 import dist as D
    for p in (abi.PREC_3XTF32, abi.PREC_TF32):
        cfg = abi.default_config(precision=p)
        assert not D.needs_agreement(cfg)
        assert D.resolve_precision(cfg, False, False).precision == p


def _c5_worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from paper_2205_08115_b200 import dist as D
    from oracle.bindings import Oracle
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b0, b1 = D.batch_range(total, rank, world)
    o = Oracle("port")
    objs = []
    for k in range(b0, b1):
        inst = I.config5_problem(k, n=24)
        cfg = abi.default_config(rho=0.1, max_iters=15, rel_tol=1e-30, quiet=1)
        r = o.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu)
        objs.append(r.trace[-1]["objective"])
    sizes = [None] * world
    dist.all_gather_object(sizes, (b0, b1, objs))
    q.put((rank, sizes))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 7), (3, 8)])
def test_c5_partition_across_ranks(world, total):
    """Config 5 across ranks (bench.py c5, no communication): the ranges tile
    the batch exactly once and the gathered per-problem results equal the
    single-process ones, in problem order."""
    from oracle.bindings import Oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c5_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = sorted(out[0], key=lambda t: t[0])
    assert parts[0][0] == 0 and parts[-1][1] == total
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    gathered = [v for _, _, objs in parts for v in objs]
    o = Oracle("port")
    want = []
    for k in range(total):
        inst = I.config5_problem(k, n=24)
        r = o.solve(abi.default_config(rho=0.1, max_iters=15, rel_tol=1e-30, quiet=1),
                    inst.dx, inst.dy, inst.mu, inst.nu)
        want.append(r.trace[-1]["objective"])
    assert gathered == want
