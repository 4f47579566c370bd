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
from paper_2205_08115_b200 import instances as I

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
}


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
                        t["rel_change"], t["phase"]] for t in r.trace])
        cfg_vec = np.array([getattr(cfg, f) for f, _ in abi.Config._fields_], dtype=np.float64)
        np.savez_compressed(os.path.join(out, name + ".npz"), dx=inst.dx, dy=inst.dy, mu=inst.mu,
                            nu=inst.nu, final=r.final, trace=tr, config=cfg_vec,
                            converged=r.converged, iterations=r.iterations_used)
        print(name, r.iterations_used, r.converged, r.trace[-1]["objective"])


if __name__ == "__main__":
    main()
