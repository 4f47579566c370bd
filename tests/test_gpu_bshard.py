"""Row-sharded eBPG / BPG / hBPG (csrc/bregman.cu sharded mode, dist.py
run_bregman_sharded) against the CPU oracle: P = 2 / 3 shard engines on one
GPU with an in-order emulated all-gather, and the public NCCL entry at
world 1.  Same bounds as the single-GPU Bregman tests."""
import numpy as np
import pytest

from paper_2205_08115_b200 import abi, dist
from harness import instances as I

pytestmark = pytest.mark.gpu


def _run(inst, world, **over):
    import torch
    kw = dict(rel_tol=1e-30, quiet=1)
    kw.update(over)
    cfg = abi.default_config(**kw)
    t = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float32, device="cuda")
    stream = torch.cuda.Stream()
    shards = dist.bregman_shards_from_dense(cfg, t(inst.dx), t(inst.dy), inst.mu, inst.nu, world,
                                            stream=stream)
    try:
        outs = dist.run_bregman_sharded(shards, dist.EmuComm(), cfg.max_iters)
    finally:
        for s in shards:
            s.close()
    return outs, cfg


def _check(outs, o):
    a = outs[0]
    for b in outs[1:]:  # replicated: every rank returns the same coupling and trace
        assert np.array_equal(a["final"], b["final"])
        assert [r.objective for r in a["trace"]] == [r.objective for r in b["trace"]]
    assert a["iterations_used"] == o.iterations_used
    assert np.abs(a["final"] - o.final).max() <= 1e-4 * np.abs(o.final).max()
    obj, ref = a["trace"][-1].objective, o.trace[-1]["objective"]
    assert abs(obj - ref) <= 1e-5 * abs(ref)
    assert [r.phase for r in a["trace"]] == [t["phase"] for t in o.trace]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("algo,over", [
    ("hbpg", dict(algorithm=abi.HBPG, epsilon_reg=0.1, step=5.0, inner_iters=10, switch_iters=4,
                  max_iters=9)),
    ("ebpg", dict(algorithm=abi.EBPG, epsilon_reg=0.1, inner_iters=10, max_iters=6)),
    ("bpg", dict(algorithm=abi.BPG, step=5.0, inner_iters=10, max_iters=6, perturbation=0.01)),
])
def test_sharded_bregman_matches_oracle(gpu, port, world, algo, over):
    inst = I.config1(seed=5, n=200)
    outs, cfg = _run(inst, world, **over)
    o = port.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu)
    assert o.code == 0, o.message
    _check(outs, o)


def test_sharded_hbpg_empty_ranks(gpu, port):
    # n = 100 over 4 ranks: 64-row shards, so ranks 2 and 3 own no rows.
    inst = I.config1(seed=9, n=100)
    outs, cfg = _run(inst, 4, algorithm=abi.HBPG, epsilon_reg=0.1, step=5.0, inner_iters=10,
                     switch_iters=2, max_iters=5)
    o = port.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu)
    _check(outs, o)


def test_sharded_hbpg_weighted_d_3xtf32(gpu, port):
    # Euclidean D: AUTO resolves to 3xTF32 (dist.resolve_precision).
    g = I.config2(seed=4, n=150, m=120)
    outs, cfg = _run(g, 2, algorithm=abi.HBPG, epsilon_reg=0.1, step=5.0, inner_iters=10,
                     switch_iters=3, max_iters=6)
    o = port.solve(cfg, g.dx, g.dy, g.mu, g.nu)
    _check(outs, o)


def test_sharded_bregman_errors(gpu):
    inst = I.config1(seed=2, n=96)
    with pytest.raises(abi.NumericalInstabilityError, match="exp overflow; reduce step"):
        _run(inst, 2, algorithm=abi.BPG, step=1e7, inner_iters=5, max_iters=5)


def test_sharded_hbpg_stop_rule(gpu, port):
    inst = I.config1(seed=7, n=120)
    outs, cfg = _run(inst, 2, algorithm=abi.HBPG, epsilon_reg=0.1, step=5.0, inner_iters=20,
                     switch_iters=5, max_iters=300, rel_tol=1e-4)
    o = port.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu)
    assert outs[0]["converged"] == o.converged
    # fp32 iterates cannot resolve the last fp64 digits: never earlier.
    assert outs[0]["iterations_used"] >= o.iterations_used


def test_solve_bregman_sharded_nccl_world1(gpu, port):
    import os
    import socket
    import torch
    import torch.distributed as tdist
    inst = I.config1(seed=8, n=160)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port_no = sk.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = abi.default_config(algorithm=abi.HBPG, epsilon_reg=0.1, step=5.0, inner_iters=10,
                                 switch_iters=3, max_iters=6, rel_tol=1e-30, quiet=1)
        r = dist.solve_bregman_sharded(cfg, inst.dx, inst.dy, inst.mu, inst.nu, tdist, 0, 1, 0)
    finally:
        tdist.destroy_process_group()
    o = port.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu)
    _check([r], o)
