"""Row-sharded multi-GPU BAPG orchestration.

One process per GPU (torchrun).  Each rank owns a contiguous block of rows of
π, w and D_X; D_Y is replicated.  The device work runs in ``libgwb.so``
(``gwb_shard_*``, csrc/shard.cu); this module owns the communication
buffers as torch tensors and issues the collectives between the phases on
the shard's CUDA stream, so NCCL (NVLink/NVSwitch) transfers are ordered
with the kernels without host synchronisation:

  per iteration   phase 0 · all-gather(Vᵀ) · phase 1 · phase 2 ·
                  all-gather(Vᵀ) · phase 3 · all-gather(col stats) · phase 4 ·
                  all-reduce-sum(diag) · all-reduce-max(err) · phase 5
  after the loop  phase 6 · all-gather(Vᵀ) · phase 7 · all-reduce(diag, err) ·
                  phase 8

`run_sharded` drives any list of shard engines with any `Comm`: real ranks
(`TorchComm`, one local shard), several virtual ranks on one GPU
(`EmuComm`, used by the GPU tests — there is only one GPU per box here), or
the CPU mirror used by the gloo tests (tests/shard_mirror.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional

from . import abi

KBLOCK_ROWS = 64  # shard rows are padded to a multiple of the bf16 k-block


@dataclass
class ShardPlan:
    """Row ownership, identical to ShardEngine (csrc/shard.cu)."""

    n: int
    world: int

    @property
    def rows_per_shard(self) -> int:
        r = -(-self.n // self.world)
        return -(-r // KBLOCK_ROWS) * KBLOCK_ROWS

    def row_begin(self, rank: int) -> int:
        return rank * self.rows_per_shard

    def rows_valid(self, rank: int) -> int:
        return max(0, min(self.rows_per_shard, self.n - self.row_begin(rank)))


_P = C.c_void_p
_I64P = C.POINTER(C.c_int64)
_I32P = C.POINTER(C.c_int32)
_ST = C.POINTER(abi.Status)
_SIGS = {
    "gwb_shard_create": (C.c_int32, [C.POINTER(abi.Config), C.c_int64, C.c_int64, C.c_int32,
                                     C.c_int32, C.c_int32, _P, C.POINTER(_P), _ST]),
    "gwb_shard_layout": (C.c_int32, [_P, _I64P, _I64P, _I64P, _I32P, _I32P, _I64P, _I64P, _ST]),
    "gwb_shard_set_comm": (C.c_int32, [_P, _P, _P, _P, _P, _ST]),
    "gwb_shard_load_device": (C.c_int32, [_P, _P, C.c_int64, _P, C.c_int64, _P, _P, _ST]),
    "gwb_shard_set_iterate_bound": (C.c_int32, [_P, C.c_double, _ST]),
    "gwb_shard_set_marginals64": (C.c_int32, [_P, _P, _P, _ST]),
    "gwb_shard_reset": (C.c_int32, [_P, _ST]),
    "gwb_shard_phase": (C.c_int32, [_P, C.c_int32, _ST]),
    "gwb_shard_stream": (C.c_int32, [_P, C.POINTER(_P), _ST]),
    "gwb_shard_launches": (C.c_int32, [_P, _I64P]),
    "gwb_shard_gemm2_chunk": (C.c_int32, [_P, C.c_int32, C.c_int32, _ST]),
    "gwb_shard_status": (C.c_int32, [_P, _I32P, _I32P, _I32P, _I32P, _I32P, _I32P, _ST]),
    "gwb_shard_finish": (C.c_int32, [_P, _ST]),
    "gwb_shard_records": (C.c_int32, [_P, C.c_int32, C.POINTER(abi.Record), _ST]),
    "gwb_shard_rows": (C.c_int32, [_P, _P, _P, _ST]),
    "gwb_shard_destroy": (C.c_int32, [_P]),
    "gwb_bshard_create": (C.c_int32, [C.POINTER(abi.Config), C.c_int64, C.c_int64, C.c_int32,
                                      C.c_int32, C.c_int32, _P, C.POINTER(_P), _ST]),
    "gwb_bshard_layout": (C.c_int32, [_P, _I64P, _I64P, _I64P, _I64P, _I64P, _I32P, _I32P, _I64P,
                                      _ST]),
    "gwb_bshard_set_comm": (C.c_int32, [_P, _P, _P, _ST]),
    "gwb_bshard_load_device": (C.c_int32, [_P, _P, C.c_int64, _P, C.c_int64, _P, _P, _ST]),
    "gwb_bshard_phase": (C.c_int32, [_P, C.c_int32, C.c_int32, _ST]),
    "gwb_bshard_status": (C.c_int32, [_P, _I32P, _I32P, _I32P, _I32P, _ST]),
    "gwb_bshard_stream": (C.c_int32, [_P, C.POINTER(_P), _ST]),
    "gwb_bshard_finish": (C.c_int32, [_P, _P, C.POINTER(abi.Record), C.c_int32, _I32P, _I32P,
                                      _I32P, _ST]),
    "gwb_bshard_destroy": (C.c_int32, [_P]),
}


def _lib():
    lib = abi.load()
    if not getattr(lib, "_shard_ready", False):
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        lib._shard_ready = True
    return lib


def _check(st: abi.Status):
    abi.raise_for(st)


class GpuShard:
    """One rank's ShardEngine plus its torch-owned communication buffers."""

    def __init__(self, cfg: abi.Config, n: int, m: int, rank: int, world: int,
                 device: int = 0, stream=None):
        import torch
        self.torch = torch
        self.lib = _lib()
        self.n, self.m, self.rank, self.world = n, m, rank, world
        st = abi.Status()
        self.h = _P()
        sp = None if stream is None else stream.cuda_stream
        self.lib.gwb_shard_create(C.byref(cfg), n, m, rank, world, device, sp, C.byref(self.h),
                                  C.byref(st))
        _check(st)
        rps, rb, rv = C.c_int64(), C.c_int64(), C.c_int64()
        pl, es, vb, sb = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64()
        self.lib.gwb_shard_layout(self.h, C.byref(rps), C.byref(rb), C.byref(rv), C.byref(pl),
                                  C.byref(es), C.byref(vb), C.byref(sb), C.byref(st))
        _check(st)
        self.rows_per_shard, self.row_begin, self.rows_valid = rps.value, rb.value, rv.value
        self.planes, self.elem_bytes = pl.value, es.value
        dev = torch.device("cuda", device)
        self.vt = torch.zeros(vb.value, dtype=torch.uint8, device=dev)
        self.stats = torch.zeros(world * 3 * m, dtype=torch.float64, device=dev)
        self.diag = torch.zeros(8, dtype=torch.float64, device=dev)
        self.err = torch.zeros(8, dtype=torch.float64, device=dev)
        self.lib.gwb_shard_set_comm(self.h, self.vt.data_ptr(), self.stats.data_ptr(),
                                    self.diag.data_ptr(), self.err.data_ptr(), C.byref(st))
        _check(st)
        sp = _P()
        self.lib.gwb_shard_stream(self.h, C.byref(sp), C.byref(st))
        self.stream = torch.cuda.ExternalStream(sp.value, device=dev)
        self.max_iters = cfg.max_iters
        self.precision = cfg.precision

    def load(self, dx_rows, dy, mu_rows, nu, x_max=None, mu64=None, nu64=None):
        """Device fp32 tensors: dx_rows (rows_valid × n, any leading dim),
        dy (m × m), mu_rows (rows_valid), nu (m).  f16x2 chains also need
        x_max = max(max μ, max ν) over ALL ranks (the iterate bound every
        rank must agree on, gwb_shard_set_iterate_bound).  `mu64` (this
        rank's rows) / `nu64` (all m): the exact host fp64 marginals the fp64
        iterates are projected onto (default: the fp32 device values)."""
        st = abi.Status()
        if self.precision == abi.PREC_F16X2:
            if x_max is None:
                raise ValueError("f16x2 shard: pass x_max = max(max mu, max nu) over all ranks")
            self.lib.gwb_shard_set_iterate_bound(self.h, float(x_max), C.byref(st))
            _check(st)
        self.torch.cuda.synchronize()
        self.lib.gwb_shard_load_device(self.h, dx_rows.data_ptr(), dx_rows.stride(0),
                                       dy.data_ptr(), dy.stride(0), mu_rows.data_ptr(),
                                       nu.data_ptr(), C.byref(st))
        _check(st)
        if mu64 is not None and nu64 is not None:
            import numpy as np
            self._mu64 = np.ascontiguousarray(mu64, dtype=np.float64)
            self._nu64 = np.ascontiguousarray(nu64, dtype=np.float64)
            self.lib.gwb_shard_set_marginals64(self.h, self._mu64.ctypes.data, self._nu64.ctypes.data,
                                               C.byref(st))
            _check(st)

    def reset(self):
        st = abi.Status()
        self.lib.gwb_shard_reset(self.h, C.byref(st))
        _check(st)

    def phase(self, k: int):
        st = abi.Status()
        self.lib.gwb_shard_phase(self.h, k, C.byref(st))
        _check(st)

    def status(self) -> dict:
        st = abi.Status()
        v = [C.c_int32() for _ in range(6)]
        self.lib.gwb_shard_status(self.h, *[C.byref(x) for x in v], C.byref(st))
        _check(st)
        keys = ("done", "iter", "flags", "converged", "err_iter", "zero_index")
        return {k: x.value for k, x in zip(keys, v)}

    def gemm2_chunk(self, src: int, tail: bool = False):
        st = abi.Status()
        self.lib.gwb_shard_gemm2_chunk(self.h, src, 1 if tail else 0, C.byref(st))
        _check(st)

    def launches(self) -> int:
        v = C.c_int64()
        self.lib.gwb_shard_launches(self.h, C.byref(v))
        return v.value

    def finish(self):
        st = abi.Status()
        self.lib.gwb_shard_finish(self.h, C.byref(st))
        _check(st)

    def records(self, count: int):
        st = abi.Status()
        out = (abi.Record * max(count, 1))()
        self.lib.gwb_shard_records(self.h, count, out, C.byref(st))
        _check(st)
        return list(out[:count])

    def rows(self, out_pi=None, out_w=None):
        """This rank's rows of π and w (fp64, rows_valid × m), into the
        caller's arrays when given (e.g. page-locked, allocated once)."""
        import numpy as np
        st = abi.Status()
        shape = (self.rows_valid, self.m)
        pi = out_pi if out_pi is not None else np.empty(shape)
        w = out_w if out_w is not None else np.empty(shape)
        for a in (pi, w):
            if a.shape != shape or a.dtype != np.float64 or not a.flags.c_contiguous:
                raise ValueError(f"rows: output must be a C-contiguous float64 array of shape {shape}")
        self.lib.gwb_shard_rows(self.h, pi.ctypes.data, w.ctypes.data, C.byref(st))
        _check(st)
        return pi, w

    def close(self):
        if self.h:
            self.lib.gwb_shard_destroy(self.h)
            self.h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class BregShard:
    """One rank's row-sharded eBPG / BPG / hBPG engine (csrc/bregman.cu) with
    its torch-owned exchange buffers: `vt` (the Vᵀ gather buffer, as
    GpuShard) and `g` (G, padded_rows × ld fp32; rank r's rows are block r)."""

    def __init__(self, cfg: abi.Config, n: int, m: int, rank: int, world: int,
                 device: int = 0, stream=None):
        import torch
        self.torch = torch
        self.lib = _lib()
        self.n, self.m, self.rank, self.world = n, m, rank, world
        self.max_iters = cfg.max_iters
        st = abi.Status()
        self.h = _P()
        sp = None if stream is None else stream.cuda_stream
        self.lib.gwb_bshard_create(C.byref(cfg), n, m, rank, world, device, sp, C.byref(self.h),
                                   C.byref(st))
        _check(st)
        v = [C.c_int64() for _ in range(5)]
        pl, es, vb = C.c_int32(), C.c_int32(), C.c_int64()
        self.lib.gwb_bshard_layout(self.h, *[C.byref(x) for x in v], C.byref(pl), C.byref(es),
                                   C.byref(vb), C.byref(st))
        _check(st)
        self.rows_per_shard, self.row_begin, self.rows_valid, self.padded_rows, self.ld = \
            (x.value for x in v)
        self.planes, self.elem_bytes = pl.value, es.value
        dev = torch.device("cuda", device)
        self.vt = torch.zeros(vb.value, dtype=torch.uint8, device=dev)
        self.g = torch.zeros(self.padded_rows * self.ld, dtype=torch.float32, device=dev)
        self.lib.gwb_bshard_set_comm(self.h, self.vt.data_ptr(), self.g.data_ptr(), C.byref(st))
        _check(st)
        spp = _P()
        self.lib.gwb_bshard_stream(self.h, C.byref(spp), C.byref(st))
        self.stream = torch.cuda.ExternalStream(spp.value, device=dev)

    def load(self, dx_rows, dy, mu, nu):
        """dx_rows / dy: device fp32 tensors (rows_valid × n, m × m); mu, nu:
        host fp64 arrays (full length)."""
        import numpy as np
        st = abi.Status()
        self.torch.cuda.synchronize()
        mu = np.ascontiguousarray(mu, dtype=np.float64)
        nu = np.ascontiguousarray(nu, dtype=np.float64)
        self.lib.gwb_bshard_load_device(self.h, dx_rows.data_ptr(), dx_rows.stride(0),
                                        dy.data_ptr(), dy.stride(0), mu.ctypes.data,
                                        nu.ctypes.data, C.byref(st))
        _check(st)

    def phase(self, k: int, op: int):
        st = abi.Status()
        self.lib.gwb_bshard_phase(self.h, k, op, C.byref(st))
        _check(st)

    def status(self) -> dict:
        st = abi.Status()
        v = [C.c_int32() for _ in range(4)]
        self.lib.gwb_bshard_status(self.h, *[C.byref(x) for x in v], C.byref(st))
        _check(st)
        return dict(zip(("done", "iter", "flags", "converged"), (x.value for x in v)))

    def finish(self, want_final: bool = True) -> dict:
        import numpy as np
        st = abi.Status()
        cap = max(1, self.max_iters)
        trace = (abi.Record * cap)()
        nr, cv, used = C.c_int32(), C.c_int32(), C.c_int32()
        final = np.zeros((self.n, self.m), order="F") if want_final else None
        self.lib.gwb_bshard_finish(self.h, None if final is None else final.ctypes.data, trace, cap,
                                   C.byref(nr), C.byref(cv), C.byref(used), C.byref(st))
        _check(st)
        return {"final": final, "trace": list(trace[: nr.value]), "converged": bool(cv.value),
                "iterations_used": used.value}

    def close(self):
        if self.h:
            self.lib.gwb_bshard_destroy(self.h)
            self.h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_bregman_sharded(shards: List, comm, max_iters: int) -> List[dict]:
    """Sharded eBPG / BPG / hBPG schedule (gwb_ext.h): per outer iteration
    GEMM1 · all-gather(Vᵀ) · GEMM2 · all-gather(G) · replicated Sinkhorn and
    record; then the tail record; returns each shard's finish() result."""
    k = 0
    for k in range(1, max_iters + 1):
        for op in (0, 1, 2):
            _all_bphase(shards, k, op)
            if op == 0:
                comm.gather_vt(shards)
            elif op == 1:
                comm.gather_g(shards)
        st = shards[0].status()
        if st["flags"] or st["done"]:
            break
    st = shards[0].status()
    if not st["flags"]:
        used = st["iter"] - 1
        _all_bphase(shards, used, 3)
        comm.gather_vt(shards)
        _all_bphase(shards, used, 4)
        comm.gather_g(shards)
        _all_bphase(shards, used, 5)
    return [s.finish() for s in shards]


def _all_bphase(shards, k, op):
    for s in shards:
        s.phase(k, op)


def solve_bregman_sharded(cfg: abi.Config, dx, dy, mu, nu, dist, rank: int, world: int,
                          device: int = 0) -> dict:
    """Row-sharded eBPG / BPG / hBPG from HOST inputs (ebpg_solve /
    bpg_solve / hbpg_solve semantics, solvers.cpp:219-426) — called by every
    rank with the same arguments; `dx` only has to slice to host rows.
    The chain is sharded by rows of D_X (Vᵀ and G all-gathered over NCCL);
    the Sinkhorn scaling and the iterate are replicated, so every rank
    returns the same final coupling and trace."""
    import numpy as np
    import torch
    n, m = len(mu), len(nu)
    plan = ShardPlan(n, world)
    rb, rv = plan.row_begin(rank), plan.rows_valid(rank)
    rows = np.ascontiguousarray(dx[rb:rb + rv], dtype=np.float32).reshape(rv, n)
    if needs_agreement(cfg):
        cfg = _agree_precision(cfg, rows if rv else None, dy, dist, device)
    shard = BregShard(cfg, n, m, rank, world, device)
    try:
        dev = torch.device("cuda", device)
        if rv == 0:
            rows = np.zeros((1, n), dtype=np.float32)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)
        shard.load(t(rows), t(dy), mu, nu)
        out = run_bregman_sharded([shard], TorchComm(dist, rank, world), cfg.max_iters)[0]
    finally:
        shard.close()
    ran_bpg = cfg.algorithm == abi.BPG or any(r.phase == 2 for r in out["trace"])
    if not cfg.quiet and rank == 0 and ran_bpg and isinstance(dx, np.ndarray):
        # The BPG step-size warning (solvers.cpp:226-234), printed when a BPG
        # phase ran, as bregman_solve does; fp64 device power iteration on
        # the full host matrices.
        from . import api
        lip = api.lipschitz_bound(api.DistanceMatrix.trusted(dx), api.DistanceMatrix.trusted(dy))
        if lip > 0.0 and cfg.step > 1.0 / lip:
            import sys
            print(f"bpg: step {cfg.step:g} exceeds sigma/L_f = {1.0 / lip:g}; descent is not "
                  "guaranteed at this step size", file=sys.stderr)
    return out


def bregman_shards_from_dense(cfg: abi.Config, dx, dy, mu, nu, world: int, device=0,
                              stream=None) -> List[BregShard]:
    """Sharded Bregman engines from full device tensors (tests / emulation);
    mu, nu host fp64."""
    import torch
    n, m = dx.shape[0], dy.shape[0]
    cfg = resolve_precision(cfg, bf16_exact(dx) and bf16_exact(dy), f16_exact(dx) and f16_exact(dy))
    shards = []
    for r in range(world):
        s = BregShard(cfg, n, m, r, world, device, stream)
        rows = dx[s.row_begin:s.row_begin + max(s.rows_valid, 1)].contiguous()
        s.load(rows, dy.contiguous(), mu, nu)
        shards.append(s)
    torch.cuda.synchronize()
    return shards


# ---------------------------------------------------------------------------
class TorchComm:
    """Collectives for one local shard per process via torch.distributed
    (NCCL on the GPU — NVLink/NVSwitch — or gloo for the CPU mirror)."""

    def __init__(self, dist, rank: int, world: int, inplace_gather: bool = True):
        self.dist, self.rank, self.world = dist, rank, world
        self.inplace = inplace_gather

    def _gather(self, buf):
        if self.inplace:
            # 1-D concatenation form (NCCL and gloo both accept it): rank r's
            # block of the flat buffer is its input, in place.
            flat = buf.view(-1)
            c = flat.numel() // self.world
            self.dist.all_gather_into_tensor(flat, flat[self.rank * c:(self.rank + 1) * c])
        else:
            view = buf.view(self.world, -1)
            parts = list(view.unbind(0))
            self.dist.all_gather(parts, view[self.rank].clone())

    def gather_vt(self, shards):
        s = shards[0]
        with _stream(s):
            self._gather(s.vt)

    def gather_stats(self, shards):
        s = shards[0]
        with _stream(s):
            self._gather(s.stats)

    def gather_g(self, shards):
        s = shards[0]
        with _stream(s):
            self._gather(s.g)

    def reduce_diag(self, shards):
        s = shards[0]
        with _stream(s):
            self.dist.all_reduce(s.diag, op=self.dist.ReduceOp.SUM)
            self.dist.all_reduce(s.err, op=self.dist.ReduceOp.MAX)

    # Chunked Vᵀ exchange for the compute/collective overlap: one broadcast
    # per source rank, all enqueued at once behind GEMM1 on the shard stream;
    # the consumer waits per chunk, so GEMM2 on landed blocks overlaps the
    # transfer of the rest.
    def start_vt_chunks(self, shards):
        s = shards[0]
        view = s.vt.view(self.world, -1)
        with _stream(s):
            return [self.dist.broadcast(view[src], src=src, async_op=True)
                    for src in range(self.world)]

    def wait_vt_chunk(self, shards, handles, src):
        s = shards[0]
        if src != self.rank:
            with _stream(s):
                handles[src].wait()

    def finish_vt_chunks(self, shards, handles):
        # Our own block was only sent: the next phase overwrites it, so the
        # stream must also be ordered after that send.
        with _stream(shards[0]):
            handles[self.rank].wait()


class EmuComm:
    """All `world` shards live in this process (one GPU, shared stream):
    collectives become device copies / reductions in rank order."""

    def gather_vt(self, shards):
        self._gather(shards, "vt")

    def gather_stats(self, shards):
        self._gather(shards, "stats")

    def gather_g(self, shards):
        self._gather(shards, "g")

    @staticmethod
    def _gather(shards, attr):
        world = len(shards)
        with _stream(shards[0]):
            views = [getattr(s, attr).view(world, -1) for s in shards]
            for r in range(world):
                for q in range(world):
                    if q != r:
                        views[q][r].copy_(views[r][r])

    def start_vt_chunks(self, shards):
        self.gather_vt(shards)  # in-order device copies: every chunk lands now
        return None

    def wait_vt_chunk(self, shards, handles, src):
        return None

    def finish_vt_chunks(self, shards, handles):
        return None

    @staticmethod
    def reduce_diag(shards):
        with _stream(shards[0]):
            total = shards[0].diag.clone()
            mx = shards[0].err.clone()
            for s in shards[1:]:
                total += s.diag
                mx = mx.maximum(s.err)
            for s in shards:
                s.diag.copy_(total)
                s.err.copy_(mx)


class _stream:
    def __init__(self, shard):
        self.s = getattr(shard, "stream", None)

    def __enter__(self):
        if self.s is not None:
            import torch
            self.ctx = torch.cuda.stream(self.s)
            self.ctx.__enter__()
        return self

    def __exit__(self, *e):
        if self.s is not None:
            self.ctx.__exit__(*e)
        return False


def _all_phase(shards, k):
    for s in shards:
        s.phase(k)


def _gemm2_overlapped(shards, comm, tail: bool):
    """Chunked exchange of Vᵀ + per-source partial GEMM2: each shard starts
    with its own block (already local), then consumes the others in the
    order their collectives were issued."""
    handles = comm.start_vt_chunks(shards)
    world = shards[0].world
    for s in shards:
        order = [s.rank] + [q for q in range(world) if q != s.rank]
        for src in order:
            comm.wait_vt_chunk([s], handles, src)
            s.gemm2_chunk(src, tail)
    comm.finish_vt_chunks(shards, handles)


def _half_a(shards, comm, overlap):
    _all_phase(shards, 0)
    if overlap:
        _gemm2_overlapped(shards, comm, False)
        _all_phase(shards, 21)
    else:
        comm.gather_vt(shards)
        _all_phase(shards, 1)


def iterate_sharded(shards: List, comm, iters: int, poll_every: int = 16,
                    overlap: bool = False) -> None:
    """Enqueue up to `iters` iterations of the phase / collective schedule.
    Every rank issues the same collectives every iteration (kernels no-op
    once done); the globally agreed `done` flag is polled every
    `poll_every` iterations (poll_every=0: never, no host synchronisation).
    overlap=True replaces each all-gather + GEMM2 by per-source collectives
    and partial GEMM2s (the transfer of later blocks overlaps the product of
    earlier ones)."""
    for it in range(1, iters + 1):
        _half_a(shards, comm, overlap)
        _all_phase(shards, 2)
        if overlap:
            _gemm2_overlapped(shards, comm, False)
            _all_phase(shards, 23)
        else:
            comm.gather_vt(shards)
            _all_phase(shards, 3)
        comm.gather_stats(shards)
        _all_phase(shards, 4)
        comm.reduce_diag(shards)
        _all_phase(shards, 5)
        if poll_every and (it % poll_every == 0 or it == iters):
            if shards[0].status()["done"]:
                break


def finish_sharded(shards: List, comm, overlap: bool = False) -> dict:
    """Objective of the last record (one more chain) and final parity."""
    st = shards[0].status()
    if not st["flags"]:
        _all_phase(shards, 6)
        if overlap:
            _gemm2_overlapped(shards, comm, True)
            _all_phase(shards, 27)
        else:
            comm.gather_vt(shards)
            _all_phase(shards, 7)
        comm.reduce_diag(shards)
        _all_phase(shards, 8)
    for s in shards:
        s.finish()
    return shards[0].status()


def run_sharded(shards: List, comm, iters: int, poll_every: int = 16,
                overlap: bool = False) -> dict:
    """Full sharded solve: iterations, then the tail record."""
    iterate_sharded(shards, comm, iters, poll_every, overlap)
    return finish_sharded(shards, comm, overlap)


def solve_sharded(cfg: abi.Config, dx, dy, mu, nu, dist, rank: int, world: int,
                  device: int = 0, poll_every: int = 16, overlap: bool = True,
                  out_pi=None, out_w=None) -> dict:
    """Row-sharded BAPG from HOST inputs — the public multi-GPU entry, called
    by every rank of a torch.distributed (NCCL) job with the same arguments.

    `dx` is anything that slices to host rows (`dx[r0:r1]`, e.g. an n×n numpy
    array, a memmap, or a lazy row builder), so a rank only materialises its
    own rows of D_X; `dy`, `mu`, `nu` are full host arrays.  The rank uploads
    its rows, runs the solve (bapg_solve semantics, solvers.cpp:138-217) and
    returns its rows of π and w (fp64; written into `out_pi` / `out_w` when
    given, rows_valid × m), the agreed trace, convergence flag and iteration
    count.  Errors raise the reference exception on every rank.
    """
    import numpy as np
    import torch
    n, m = len(mu), len(nu)
    if needs_agreement(cfg):
        # Every rank checks its own rows of D_X (and D_Y); the verdicts are
        # all-reduced (minimum), so all ranks pick the same chain.
        plan = ShardPlan(n, world)
        rb0, rv0 = plan.row_begin(rank), plan.rows_valid(rank)
        cfg = _agree_precision(cfg, np.asarray(dx[rb0:rb0 + rv0], dtype=np.float32) if rv0 else None,
                               dy, dist, device)
    shard = GpuShard(cfg, n, m, rank, world, device)
    try:
        rb, rv = shard.row_begin, shard.rows_valid
        dev = torch.device("cuda", device)
        rows = np.ascontiguousarray(dx[rb:rb + rv], dtype=np.float32).reshape(rv, n)
        if rv == 0:
            rows = np.zeros((1, n), dtype=np.float32)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)
        dx_d, dy_d = t(rows), t(dy)
        mu_d = t(np.asarray(mu)[rb:rb + max(rv, 1)] if rv else np.zeros(1))
        shard.load(dx_d, dy_d, mu_d, t(nu),
                   x_max=float(max(np.abs(np.asarray(mu)).max(), np.abs(np.asarray(nu)).max())),
                   mu64=np.asarray(mu, dtype=np.float64)[rb:rb + max(rv, 1)] if rv else np.zeros(1),
                   nu64=np.asarray(nu, dtype=np.float64))
        del dx_d, dy_d
        shard.reset()
        st = run_sharded([shard], TorchComm(dist, rank, world), cfg.max_iters, poll_every,
                         overlap)
        raise_shard_flags(st)
        used = st["iter"] - 1
        recs = shard.records(used)
        pi, w = shard.rows(out_pi, out_w)
        return {"pi_rows": pi, "w_rows": w, "row_begin": rb, "trace": recs,
                "converged": bool(st["converged"]), "iterations_used": used,
                "launches": shard.launches()}
    finally:
        shard.close()


def batch_range(total: int, rank: int, world: int):
    """Contiguous problem range [b0, b1) of `rank` when `total` independent
    problems (config 5) are partitioned over `world` ranks with no
    communication — the same split gwb_bapg_solve_batched makes across the
    devices of one process."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return total * rank // world, total * (rank + 1) // world


def raise_shard_flags(st: dict):
    """Reference error semantics from the agreed flags (solvers.cpp:164-189)."""
    f, it = st["flags"], st["err_iter"]
    if not f:
        return

    def num(detail):
        raise abi.NumericalInstabilityError(
            f"numerical instability in bapg at iteration {it}: {detail}", "bapg", it)

    if f & 1:
        num("exp overflow; increase rho")
    if f & 2:
        num(f"row {st['zero_index']} has nonpositive sum; cannot rescale")
    if f & 4:
        num("exp overflow; increase rho")
    if f & 8:
        num(f"column {st['zero_index']} has nonpositive sum; cannot rescale")
    num("non-finite iterate")


def f16_exact(t) -> bool:
    """True if every entry of the (torch or numpy) array is exact in fp16."""
    import numpy as np
    import torch
    x = t if isinstance(t, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(t, dtype=np.float32))
    x = x.float()
    return bool(torch.equal(x.to(torch.float16).float(), x))


def exact_flags(t) -> int:
    """Bit 1: exact in bf16; bit 2: exact in fp16 (the AUTO verdict ranks agree on)."""
    return (1 if bf16_exact(t) else 0) | (2 if f16_exact(t) else 0)


def bf16_exact(t) -> bool:
    """True if every entry of the (torch or numpy) array is exact in bf16."""
    import numpy as np
    import torch
    x = t if isinstance(t, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(t, dtype=np.float32))
    x = x.float()
    return bool(torch.equal(x.to(torch.bfloat16).float(), x))


def _agree_precision(cfg: abi.Config, rows, dy, dist, device: int) -> abi.Config:
    """AUTO across ranks: each rank tests its own rows of D_X (None: owns no
    rows) and D_Y for bf16 / fp16 exactness; a MIN all-reduce of the two
    verdicts makes every rank resolve the same chain."""
    import numpy as np
    import torch
    dyf = np.asarray(dy, dtype=np.float32)
    ok_bf = (rows is None or bf16_exact(rows)) and bf16_exact(dyf)
    ok_f16 = (rows is None or f16_exact(rows)) and f16_exact(dyf)
    dev = torch.device("cuda", device) if torch.cuda.is_available() else torch.device("cpu")
    flag = torch.tensor([int(ok_bf), int(ok_f16)], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    return resolve_precision(cfg, bool(flag[0].item()), bool(flag[1].item()))


def resolve_precision(cfg: abi.Config, exact: bool, f16: bool = False) -> abi.Config:
    """AUTO resolved as the single-GPU engine does: f16x2 when
    both structure matrices are exact in fp16, bf16x3 when exact in bf16,
    else 3xTF32.  With sharded D_X the exactness must be agreed by every
    rank first (each rank only sees its rows): `exact` / `f16` are those
    global verdicts."""
    p = cfg.precision
    if p == abi.PREC_AUTO:
        p = abi.PREC_F16X2 if f16 else abi.PREC_BF16X3 if exact else abi.PREC_3XTF32
    # An explicit split-plane request on a D that is not exact in its format
    # falls back as the single-GPU engine does (solver.cu prepare_d):
    # f16x2 -> bf16x3 -> 3xTF32.
    if p == abi.PREC_F16X2 and not f16:
        p = abi.PREC_BF16X3
    if p in (abi.PREC_BF16X3, abi.PREC_BF16X2) and not exact:
        p = abi.PREC_3XTF32
    if p == cfg.precision:
        return cfg
    out = abi.Config()
    C.pointer(out)[0] = cfg
    out.precision = p
    return out


def needs_agreement(cfg: abi.Config) -> bool:
    """AUTO and the split-plane chains depend on D's exactness, which each
    rank only sees for its own rows."""
    return cfg.precision in (abi.PREC_AUTO, abi.PREC_F16X2, abi.PREC_BF16X3, abi.PREC_BF16X2)


def shards_from_dense(cfg: abi.Config, dx, dy, mu, nu, world: int, ranks=None, device=0,
                      stream=None, mu64=None, nu64=None) -> List[GpuShard]:
    """Build shard engines from full device tensors (tests / emulation)."""
    import torch
    n, m = dx.shape[0], dy.shape[0]
    cfg = resolve_precision(cfg, bf16_exact(dx) and bf16_exact(dy), f16_exact(dx) and f16_exact(dy))
    x_max = float(max(mu.abs().max().item(), nu.abs().max().item()))
    shards = []
    for r in (range(world) if ranks is None else ranks):
        s = GpuShard(cfg, n, m, r, world, device, stream)
        rb, rv = s.row_begin, s.rows_valid
        rows = dx[rb:rb + max(rv, 1)].contiguous()
        murows = mu[rb:rb + max(rv, 1)].contiguous()
        s.load(rows, dy.contiguous(), murows, nu.contiguous(), x_max=x_max,
               mu64=None if mu64 is None else mu64[rb:rb + max(rv, 1)], nu64=nu64)
        shards.append(s)
    torch.cuda.synchronize()
    return shards
