"""CPU (fp64 numpy) mirror of one rank of the row-sharded eBPG / BPG / hBPG
engine (csrc/bregman.cu sharded mode) with the same exchange buffers and
phase boundaries, so `paper_2205_08115_b200.dist.run_bregman_sharded` runs
with real gloo collectives on CPU.  Phases 0/1 compute this rank's Vᵀ block
and G rows from its D_X rows; phase 2 runs the outer iteration on the
gathered G (ebpg_solve / bpg_solve, solvers.cpp:219-363, plain-domain
Sinkhorn projections.cpp:92-116).  Test infrastructure only."""
from __future__ import annotations

import numpy as np
import torch

from paper_2205_08115_b200 import abi
from paper_2205_08115_b200.dist import ShardPlan


class CpuBregShard:
    def __init__(self, cfg, dx, dy, mu, nu, rank, world):
        self.cfg, self.rank, self.world = cfg, rank, world
        self.n, self.m = dx.shape[0], dy.shape[0]
        plan = ShardPlan(self.n, world)
        self.nr = plan.rows_per_shard
        self.rb, self.rv = plan.row_begin(rank), plan.rows_valid(rank)
        self.npad = self.nr * world
        self.Dx = np.zeros((self.nr, self.npad))
        self.Dx[: self.rv, : self.n] = dx[self.rb:self.rb + self.rv]
        self.Dfull = np.asarray(dx, float)  # objective of the records only
        self.Dy = np.asarray(dy, float)
        self.mu, self.nu = np.asarray(mu, float), np.asarray(nu, float)
        self.vt = torch.zeros(world * self.m * self.nr, dtype=torch.float64)
        self.g = torch.zeros(self.npad * self.m, dtype=torch.float64)
        self.stream = None
        self.pi = np.outer(self.mu, self.nu)
        self.iter, self.done, self.flags, self.conv = 1, False, 0, False
        algo = cfg.algorithm
        self.budget1 = cfg.max_iters if algo == abi.EBPG else 0 if algo == abi.BPG else \
            min(cfg.switch_iters, cfg.max_iters)
        self.phase_now = 1 if self.budget1 >= 1 else 2
        self.used1 = 0
        self.trace = []
        self.max_iters = cfg.max_iters

    def _pad_rows(self, x):
        out = np.zeros((self.npad, self.m))
        out[: self.n] = x
        return out

    def phase(self, k, op):
        if op in (0, 3):  # this rank's Vᵀ block: (π_rows · D_Y)ᵀ
            rows = self._pad_rows(self.pi)[self.rb:self.rb + self.nr]
            self.vt.view(self.world, self.m, self.nr)[self.rank] = torch.from_numpy((rows @ self.Dy).T)
        elif op in (1, 4):  # this rank's rows of G = D_X[rows, :] · V
            vt = self.vt.view(self.world, self.m, self.nr).numpy()
            V = np.concatenate(list(vt), axis=1).T
            self.g.view(self.world, self.nr, self.m)[self.rank] = torch.from_numpy(self.Dx @ V)
        elif op == 2 and not self.done:
            G = self.g.view(self.npad, self.m).numpy()[: self.n]
            self._outer(k, G)

    def _sinkhorn(self, K):
        c = self.cfg
        for _ in range(c.inner_iters):
            K = K * (self.mu / K.sum(axis=1))[:, None]
            K = K * (self.nu / K.sum(axis=0))[None, :]
            err = max(np.abs(K.sum(axis=1) - self.mu).max(), np.abs(K.sum(axis=0) - self.nu).max())
            if err <= c.inner_tol:
                break
        return K

    def _outer(self, k, G):
        c = self.cfg
        ebpg = self.phase_now == 1
        if ebpg:
            E = (2.0 / c.epsilon_reg) * G
            K = np.exp(E - E.max())
            K = np.maximum(K, 1e-300)
            new = self._sinkhorn(K)
        else:
            E = 2.0 * c.step * G
            if E.max() > 700.0:
                self.flags, self.done = 1, True
                return
            new = self._sinkhorn(np.maximum(self.pi * np.exp(E), 1e-300))
            if c.perturbation > 0.0:
                new = (1.0 - c.perturbation) * new + c.perturbation / (self.n * self.m)
        rel = np.linalg.norm(new - self.pi) / np.linalg.norm(self.pi)
        self.pi = new
        M = self.Dfull @ new @ self.Dy
        infeas = np.linalg.norm(new.sum(axis=0) - self.nu) / self.m + \
            np.linalg.norm(new.sum(axis=1) - self.mu) / self.n
        self.trace.append(dict(objective=-(M * new).sum(), marginal_infeasibility=infeas,
                               rel_change=rel, phase=self.phase_now if c.algorithm == abi.HBPG else 0))
        self.iter = k + 1
        converged = rel <= c.rel_tol
        if ebpg and c.algorithm == abi.HBPG:
            if converged or k >= self.budget1:
                self.used1 = k
                if k < c.max_iters:
                    self.phase_now = 2
                    return
                self.conv, self.done = converged, True
                return
        if converged or k >= c.max_iters:
            self.conv, self.done = converged, True

    def status(self):
        return {"done": int(self.done), "iter": self.iter, "flags": self.flags,
                "converged": int(self.conv)}

    def finish(self):
        if self.flags:
            raise abi.NumericalInstabilityError("exp overflow; reduce step", "bpg", self.iter)
        return {"final": self.pi, "trace": self.trace, "converged": self.conv,
                "iterations_used": self.iter - 1}
