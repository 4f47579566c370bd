"""Graph inputs: gw::Graph validation (types.cpp:155-174), adjacency_distance
(tasks.cpp:167-174) and gwb_solve_graphs, which builds D on the device from
the edge list.  On the GPU the graph path must reproduce the dense-input
path bit for bit (same fp32 D, deterministic kernels)."""
import ctypes as C

import numpy as np
import pytest

import paper_2205_08115_b200 as gw
from paper_2205_08115_b200 import abi
from harness import instances as I


def test_graph_canonical_edges():
    g = gw.Graph(5, [(3, 1), (1, 3), (0, 4), (2, 0)])
    assert g.edges().tolist() == [[0, 2], [0, 4], [1, 3]]
    d = gw.adjacency_distance(g)
    assert d.size() == 5
    e = d.entries()
    assert np.array_equal(e, e.T) and e.sum() == 6 and e[1, 3] == 1.0


@pytest.mark.parametrize("n,edges,msg", [
    (0, [], "graph must have at least one node"),
    (4, [(1, 1)], "self-loop at node 1"),
    (4, [(0, 4)], r"edge \(0,4\) out of range for 4 nodes"),
    (4, [(-1, 2)], r"edge \(-1,2\) out of range for 4 nodes"),
])
def test_graph_validation_messages(n, edges, msg):
    with pytest.raises(ValueError, match=msg):
        gw.Graph(n, edges)


def _abi_graphs(n, ex, m, ey):
    lib = abi.load()
    cfg = abi.default_config(max_iters=2)
    st = abi.Status()
    ex = np.ascontiguousarray(np.asarray(ex, dtype=np.int32).reshape(-1, 2))
    ey = np.ascontiguousarray(np.asarray(ey, dtype=np.int32).reshape(-1, 2))
    u = lambda k: np.full(max(k, 1), 1.0 / max(k, 1))
    out = np.zeros(max(n * m, 1))
    i32 = C.POINTER(C.c_int32)
    d = C.POINTER(C.c_double)
    rc = lib.gwb_solve_graphs(C.byref(cfg), n, ex.ctypes.data_as(i32), len(ex), m,
                              ey.ctypes.data_as(i32), len(ey), u(n).ctypes.data_as(d),
                              u(m).ctypes.data_as(d), None, abi.OBSERVER(), None,
                              out.ctypes.data_as(d), None, None, None, 0, None, None, None,
                              C.byref(st))
    return rc, st.message.decode()


def test_cabi_graph_validation_before_device():
    # The C-ABI validates the edge lists (reference Graph messages) before
    # touching a device, so these run without a GPU.
    rc, msg = _abi_graphs(3, [(0, 0)], 3, [(0, 1)])
    assert rc == abi.ERR_INVALID and msg == "self-loop at node 0"
    rc, msg = _abi_graphs(3, [(0, 1)], 3, [(0, 7)])
    assert rc == abi.ERR_INVALID and msg == "edge (0,7) out of range for 3 nodes"
    rc, msg = _abi_graphs(0, [], 3, [])
    assert rc == abi.ERR_INVALID and msg == "graph must have at least one node"


def _pair(n=256, seed=2, q=0.05):
    e = I.erdos_renyi(n, 0.03, seed)
    noisy = I.edge_noise(n, e, q, q, I.mix_seed(seed, 1))
    tgt, _ = I.permute_graph(n, noisy, I.mix_seed(seed, 2))
    return gw.Graph(n, e), gw.Graph(n, tgt)


@pytest.mark.gpu
@pytest.mark.parametrize("algorithm", ["bapg", "hbpg"])
def test_graph_path_matches_dense_path(gpu, port, algorithm):
    gx, gy = _pair()
    n = gx.num_nodes()
    u = gw.ProbabilityVector(np.full(n, 1.0 / n))
    extra = dict(switch_iters=10, inner_iters=10, epsilon_reg=0.1) if algorithm == "hbpg" else {}
    cfg = gw.SolverConfig(algorithm=algorithm, rho=0.1, max_iters=25, rel_tol=1e-30, quiet=True,
                          **extra)
    a = gw.solve(gw.adjacency_distance(gx), gw.adjacency_distance(gy), u, u, cfg)
    dx = gw.adjacency_distance(gx).entries()
    dy = gw.adjacency_distance(gy).entries()
    b = gw.solve(gw.DistanceMatrix(dx), gw.DistanceMatrix(dy), u, u, cfg)
    assert np.array_equal(a.final_coupling.entries(), b.final_coupling.entries())
    assert [r.objective for r in a.trace] == [r.objective for r in b.trace]
    o = port.solve(cfg.to_abi(), dx, dy, u.weights(), u.weights())
    assert abs(a.trace[-1].objective - o.trace[-1]["objective"]) <= 1e-5 * abs(o.trace[-1]["objective"])
