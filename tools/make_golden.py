"""Generate tests/golden/*.npz from the REFERENCE's own solver code
(oracle/_ref: the reference TUs built against eigen_lite, OpenBLAS off so
the GEMM is the plain loop).  Run in the container that has /root/reference;
the fixtures travel with the repo so the GPU box can check against them."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from oracle.bindings import Oracle
from paper_2205_08115_b200 import abi
from harness import instances as I

CASES = {
    "bapg_er64": (lambda: I.config1(seed=11, n=64), dict(algorithm=abi.BAPG, rho=0.1, max_iters=60)),
    "bapg_gmm48x40": (lambda: I.config2(seed=12, n=48, m=40), dict(algorithm=abi.BAPG, rho=0.05, max_iters=40)),
    "bapg_sbm60k5": (lambda: I.config3(seed=13, n=60, k=5), dict(algorithm=abi.BAPG, rho=0.5, max_iters=40)),
    "bapg_ba80_stop": (lambda: I.alignment_instance(I.barabasi_albert(80, 3, 14), 80, 0.05, 14, "ba80", {}),
                       dict(algorithm=abi.BAPG, rho=0.1, max_iters=2000, rel_tol=1e-6)),
    "ebpg_er48": (lambda: I.config1(seed=15, n=48), dict(algorithm=abi.EBPG, epsilon_reg=0.1, max_iters=12, inner_iters=10)),
    "bpg_er48": (lambda: I.config1(seed=16, n=48), dict(algorithm=abi.BPG, step=5.0, max_iters=10, inner_iters=10)),
    "hbpg_er48": (lambda: I.config1(seed=17, n=48), dict(algorithm=abi.HBPG, epsilon_reg=0.1, step=5.0,
                                                         inner_iters=10, switch_iters=5, max_iters=12)),
    # quadratic geometry (euclid_project) and the per-record Luo-Tseng residual
    "bapg_quad_gmm40x32": (lambda: I.config2(seed=18, n=40, m=32),
                           dict(algorithm=abi.BAPG, geometry=abi.QUADRATIC, rho=2.0, max_iters=25)),
    "bapg_er40_residual": (lambda: I.config1(seed=19, n=40),
                           dict(algorithm=abi.BAPG, rho=0.5, max_iters=6, record_residual=1)),
    "hbpg_er36_residual": (lambda: I.config1(seed=20, n=36),
                           dict(algorithm=abi.HBPG, epsilon_reg=0.1, step=5.0, inner_iters=10,
                                switch_iters=3, max_iters=6, record_residual=1)),
}


def leaf_fixtures(ref, out):
    """Leaves off the solver path: luo_tseng_residual / dykstra_project
    (diagnostics.cpp:33-42, projections.cpp:165-187) and write_coupling_csv
    (io.cpp:183-193), computed by the reference build."""
    rng = np.random.default_rng(21)
    n, m = 40, 30
    dx = I.adjacency(n, I.erdos_renyi(n, 0.2, 21))
    dy = I.adjacency(m, I.erdos_renyi(m, 0.2, 22))
    mu = rng.uniform(0.5, 1.5, n)
    nu = rng.uniform(0.5, 1.5, m)
    mu, nu = mu / mu.sum(), nu / nu.sum()
    pi = np.asfortranarray(np.outer(mu, nu) * rng.uniform(0.5, 1.5, (n, m)))
    rc, res, msg = ref.luo_tseng_residual(dx, dy, pi, mu, nu)
    assert rc == 0, msg
    rc, proj, msg = ref.dykstra_project(3.0 * pi, mu, nu)
    assert rc == 0, msg
    np.savez_compressed(os.path.join(out, "leaf_residual_er40x30.npz"), dx=dx, dy=dy, mu=mu, nu=nu,
                        pi=pi, residual=res, dykstra_in=3.0 * pi, dykstra_out=proj)
    print("leaf_residual_er40x30", res)
    a = rng.standard_normal((12, 9)) * 10.0 ** rng.integers(-320, 300, (12, 9))
    a.flat[:10] = [0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1e16, 1e17, 1e-4, 1e-5]
    k = rng.integers(4 * 10**15, 9 * 10**15, 8) | 1
    a.flat[10:18] = k.astype(np.float64) / 4.0  # exact 17th-digit ties
    a = np.asfortranarray(a)
    text = ref.format_coupling_csv(a)
    np.savez_compressed(os.path.join(out, "leaf_csv_mixed12x9.npz"), a=a,
                        text=np.frombuffer(text, dtype=np.uint8))
    print("leaf_csv_mixed12x9", len(text), "bytes")


def main():
    ref = Oracle("reference", blas=False)
    out = os.path.join(ROOT, "tests", "golden")
    os.makedirs(out, exist_ok=True)
    for name, (make, over) in CASES.items():
        inst = make()
        kw = dict(rel_tol=1e-30, quiet=1)
        kw.update(over)
        cfg = abi.default_config(**kw)
        r = ref.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu)
        assert r.code == 0, r.message
        tr = np.array([[t["iter"], t["objective"], t["marginal_infeasibility"], t["split_gap"],
                        t["rel_change"], t["phase"],
                        np.nan if t.get("residual") is None else t["residual"]] for t in r.trace])
        cfg_vec = np.array([getattr(cfg, f) for f, _ in abi.Config._fields_], dtype=np.float64)
        np.savez_compressed(os.path.join(out, name + ".npz"), dx=inst.dx, dy=inst.dy, mu=inst.mu,
                            nu=inst.nu, final=r.final, trace=tr, config=cfg_vec,
                            converged=r.converged, iterations=r.iterations_used)
        print(name, r.iterations_used, r.converged, r.trace[-1]["objective"])
    leaf_fixtures(ref, out)


if __name__ == "__main__":
    main()
