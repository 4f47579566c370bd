"""CPU (fp64 numpy) mirror of one rank of the row-sharded BAPG
(csrc/shard.cu), with the same buffer layouts, phase boundaries and
collective schedule, so `paper_2205_08115_b200.dist.run_sharded` can be
exercised with real gloo collectives on CPU (world_size ≥ 2).  Test
infrastructure: it checks the sharding plan, the gather layout, the
rank-ordered column merge and the agreed stop/error decision; the CUDA
phases themselves are checked against the oracle in tests/test_gpu_dist.py.
"""
from __future__ import annotations

import numpy as np
import torch

from paper_2205_08115_b200.dist import ShardPlan


class CpuShard:
    def __init__(self, dx, dy, mu, nu, rho, rank, world, max_iters, rel_tol):
        self.n, self.m = dx.shape[0], dy.shape[0]
        self.rank, self.world = rank, world
        plan = ShardPlan(self.n, world)
        self.nr = plan.rows_per_shard
        self.rb, self.rv = plan.row_begin(rank), plan.rows_valid(rank)
        self.rho, self.rel_tol, self.max_iters = rho, rel_tol, max_iters
        kpad = self.nr * world
        self.Dx = np.zeros((self.nr, kpad))
        self.Dx[: self.rv, : self.n] = dx[self.rb:self.rb + self.rv]
        self.Dy = np.array(dy, dtype=float)
        self.mu = np.asarray(mu, float)[self.rb:self.rb + self.rv]
        self.nu = np.asarray(nu, float)
        self.vt = torch.zeros(world * 1 * self.m * self.nr, dtype=torch.float64)
        self.stats = torch.zeros(world * 3 * self.m, dtype=torch.float64)
        self.diag = torch.zeros(8, dtype=torch.float64)
        self.err = torch.zeros(8, dtype=torch.float64)
        self.stream = None
        self.records = {}

    def reset(self):
        self.W = np.zeros((self.nr, self.m))
        self.W[: self.rv] = np.outer(self.mu, self.nu)
        self.P = np.zeros((self.nr, self.m))
        self.iter, self.done, self.gdone, self.flags, self.conv = 1, False, False, 0, False
        self.err_iter, self.zero_index = 0, 0

    # -- helpers ------------------------------------------------------------
    def _slot(self):
        return self.vt.view(self.world, self.m, self.nr)[self.rank].numpy()

    def _G(self):
        vt = self.vt.view(self.world, self.m, self.nr).numpy()
        V = np.concatenate(list(vt), axis=1).T          # (world·nr) × m
        return self.Dx @ V

    def _rec(self, k):
        return self.records.setdefault(k, {})

    def gemm2_chunk(self, src, tail=False):
        """Partial GEMM2 over the Vᵀ block of rank `src` (ShardEngine::gemm2_chunk)."""
        if (self.flags if tail else self.done):
            return
        chunk = self.vt.view(self.world, self.m, self.nr).numpy()[src]  # m × nr
        part = self.Dx[:, src * self.nr:(src + 1) * self.nr] @ chunk.T
        self.Gacc = part if src == self.rank else self.Gacc + part

    # -- phases (csrc/shard.cu ShardEngine::phase) ----------------------------
    def phase(self, ph):
        rv = self.rv
        chunked = ph >= 20
        if chunked:
            ph -= 20
        full_G = (lambda: self.Gacc) if chunked else self._G
        if ph in (0, 6):
            if ph == 0 and self.done:
                return
            self._slot()[:] = self.Dy @ self.W.T
        elif ph in (1, 7):
            if ph == 1 and self.done:
                return
            G = full_G()[:rv]
            W = self.W[:rv]
            self.row_gw = float(np.sum(G * W))
            self.row_dev = float(np.sum((W.sum(1) - self.mu) ** 2))
            if ph == 7:
                self._write_diag(tail=True)
                return
            E = G / self.rho
            rmax = E.max(1) if rv else np.zeros(0)
            T = W * np.exp(E - rmax[:, None])
            S = T.sum(1)
            if np.any(rmax > 700):
                self.flags |= 1
            bad = np.nonzero(~(S > 0))[0]
            if bad.size:
                self.flags |= 2
                self.zero_index = int(bad[0])
            self.P[:rv] = (self.mu / S)[:, None] * T
            if self.flags:
                self.done = True
        elif ph == 2:
            if self.done:
                return
            self._slot()[:] = self.Dy @ self.P.T
        elif ph == 3:
            if self.done:
                return
            G = full_G()[:rv]
            self.G = G
            E = G / self.rho
            P = self.P[:rv]
            st = self.stats.view(self.world, 3, self.m)[self.rank].numpy()
            if rv:
                mx = E.max(0)
                st[0] = mx
                st[1] = np.sum(P * np.exp(E - mx), 0)
                st[2] = P.sum(0)
            else:
                st[0], st[1], st[2] = -np.inf, 0.0, 0.0
        elif ph == 4:
            if not self.done:
                stats = self.stats.view(self.world, 3, self.m).numpy()
                mx = np.full(self.m, -np.inf)
                s = np.zeros(self.m)
                p = np.zeros(self.m)
                for r in range(self.world):  # rank order
                    cm, cs = stats[r, 0], stats[r, 1]
                    valid = cm > -np.inf
                    newmx = np.where(valid, np.maximum(mx, cm), mx)
                    with np.errstate(invalid="ignore"):
                        old = np.where(np.isfinite(mx), np.exp(mx - newmx), 0.0)
                        s = np.where(valid, s * old + cs * np.exp(cm - newmx), s)
                    mx = newmx
                    p += stats[r, 2]
                if np.any(mx > 700):
                    self.flags |= 4
                bad = np.nonzero(~(s > 0))[0]
                if bad.size:
                    self.flags |= 8
                    self.zero_index = int(bad[0])
                self.col_dev = float(np.sum((p - self.nu) ** 2))
                if not self.flags:
                    G = self.G
                    E = G / self.rho
                    P = self.P[:rv]
                    Wn = np.zeros_like(self.W)
                    Wn[:rv] = (self.nu / s)[None, :] * P * np.exp(E - mx[None, :])
                    W = self.W[:rv]
                    self.cw = [float(np.sum(G * Wn[:rv])), float(np.sum((P - Wn[:rv]) ** 2)),
                               float(np.sum((Wn[:rv] - W) ** 2)), float(np.sum(W ** 2)),
                               float(np.sum(G * P))]
                    self.W_new = Wn
                else:
                    self.done = True
            self._write_diag(tail=False)
        elif ph in (5, 8):
            self._finalize(tail=ph == 8)

    def _write_diag(self, tail):
        d = np.zeros(8)
        active = (self.flags == 0) if tail else not self.gdone
        if active:
            d[0], d[1] = self.row_gw, self.row_dev
            if not tail and not self.flags:
                d[2:7] = self.cw
                if self.rank == 0:
                    d[7] = self.col_dev
        self.diag[:] = torch.from_numpy(d)
        f = self.flags if active else 0
        e = [float(bool(f & b)) for b in (1, 2, 4, 8, 16)]
        e += [-(self.rb + self.zero_index) if f & 2 else -1e18,
              -self.zero_index if f & 8 else -1e18, 0.0]
        self.err[:] = torch.tensor(e, dtype=torch.float64)

    def _finalize(self, tail):
        d, e = self.diag.numpy(), self.err.numpy()
        if self.gdone:
            self.done = True
            if not tail or self.flags:
                return
        if tail:
            k = self.iter - 1
            self._rec(k).update(mw_w=d[0], row_sq=d[1])
            return
        k = self.iter
        gflags = sum(b for b, v in zip((1, 2, 4, 8, 16), e[:5]) if v > 0.5)
        if gflags:
            self.flags = gflags
            self.zero_index = int(-e[5] if gflags & 2 else -e[6])
            self.err_iter = k
            self.done = self.gdone = True
            return
        if k >= 2:
            self._rec(k - 1).update(mw_w=d[0], row_sq=d[1])
        self._rec(k).update(mpi_w=d[2], split_sq=d[3], diff_sq=d[4], wold_sq=d[5], mpi_pi=d[6],
                            col_sq=d[7])
        self.iter = k + 1
        self.W = self.W_new
        rel = np.sqrt(d[4]) / np.sqrt(d[5])
        if rel <= self.rel_tol:  # the reference rule (fp64 shard iterates, shard.cu)
            self.conv = True
            self.done = self.gdone = True

    def status(self):
        return {"done": int(self.done), "iter": self.iter, "flags": self.flags,
                "converged": int(self.conv), "err_iter": self.err_iter,
                "zero_index": self.zero_index}

    def finish(self):
        pass

    def trace(self, count):
        out = []
        for k in range(1, count + 1):
            r = self.records[k]
            out.append(dict(
                objective=-0.25 * (r["mpi_pi"] + 2 * r["mpi_w"] + r["mw_w"]),
                marginal_infeasibility=0.5 * np.sqrt(r["col_sq"]) / self.m
                + 0.5 * np.sqrt(r["row_sq"]) / self.n,
                split_gap=np.sqrt(r["split_sq"]),
                rel_change=np.sqrt(r["diff_sq"]) / np.sqrt(r["wold_sq"])))
        return out

    def rows(self):
        return self.P[: self.rv].copy(), self.W[: self.rv].copy()
