"""Instance generators (csrc/instances.cpp) against the reference's own
tasks.cpp generators: identical edge lists for the same seeds."""
import ctypes as C

import numpy as np
import pytest

from paper_2205_08115_b200 import abi
from harness import instances as I
from tests.conftest import have_ref

needs_ref = pytest.mark.skipif(not have_ref(), reason="reference build absent")


def _ref_edges(fn, *args, cap=1 << 20):
    buf = np.empty(2 * cap, dtype=np.int32)
    cnt = C.c_int64(0)
    st = abi.Status()
    fn(*args, buf.ctypes.data_as(C.POINTER(C.c_int32)), cap, C.byref(cnt), C.byref(st))
    assert st.code == 0, st.message
    return buf[: 2 * cnt.value].reshape(-1, 2)


@needs_ref
@pytest.mark.parametrize("n,m_attach,seed", [(50, 2, 1), (300, 5, 7), (1000, 3, 42)])
def test_barabasi_albert_matches_reference(n, m_attach, seed):
    from oracle.bindings import reference_generators
    lib = reference_generators()
    ref = _ref_edges(lib.gwref_gen_barabasi_albert, n, m_attach, seed)
    np.testing.assert_array_equal(I.barabasi_albert(n, m_attach, seed), ref)


@needs_ref
@pytest.mark.parametrize("n,p,seed", [(60, 0.1, 0), (400, 0.01, 3)])
def test_erdos_renyi_is_single_cluster_partition(n, p, seed):
    from oracle.bindings import reference_generators
    lib = reference_generators()
    labels = np.empty(n, dtype=np.int32)
    buf = np.empty(2 * n * n, dtype=np.int32)
    cnt = C.c_int64(0)
    st = abi.Status()
    lib.gwref_gen_gaussian_partition(n, 1, p, 0.0, seed, buf.ctypes.data_as(C.POINTER(C.c_int32)),
                                     n * n, C.byref(cnt), labels.ctypes.data_as(C.POINTER(C.c_int32)),
                                     C.byref(st))
    assert st.code == 0
    np.testing.assert_array_equal(I.erdos_renyi(n, p, seed), buf[: 2 * cnt.value].reshape(-1, 2))


@needs_ref
def test_permute_graph_matches_reference():
    from oracle.bindings import reference_generators
    lib = reference_generators()
    e = I.barabasi_albert(200, 3, 5)
    out = np.empty_like(e)
    perm = np.empty(200, dtype=np.int32)
    st = abi.Status()
    P = C.POINTER(C.c_int32)
    lib.gwref_permute_graph(200, e.ctypes.data_as(P), e.shape[0], 99, out.ctypes.data_as(P),
                            perm.ctypes.data_as(P), C.byref(st))
    got, gperm = I.permute_graph(200, e, 99)
    np.testing.assert_array_equal(gperm, perm)
    np.testing.assert_array_equal(got, out)


def test_edge_noise_counts_and_determinism():
    e = I.erdos_renyi(300, 0.05, 1)
    a = I.edge_noise(300, e, 0.05, 0.05, 9)
    b = I.edge_noise(300, e, 0.05, 0.05, 9)
    np.testing.assert_array_equal(a, b)
    k = int(np.floor(0.05 * len(e)))
    kept = set(map(tuple, e)) & set(map(tuple, a))
    assert len(kept) == len(e) - k and len(a) == len(e)
    assert np.all(a[:, 0] < a[:, 1])


def test_config_shapes():
    c3 = I.config3(n=200, k=5)
    assert c3.dx.shape == (200, 200) and c3.dy.shape == (5, 5)
    assert abs(c3.mu.sum() - 1) <= 1e-12 and np.all(c3.mu > 0)
    c2 = I.config2(n=64, m=48)
    assert c2.dx.max() == 1.0 and np.allclose(c2.dx, c2.dx.T)
    assert np.all(c2.dx.astype(np.float32) == c2.dx)
    c1 = I.config1(n=100)
    assert np.array_equal(np.sort(c1.dx.sum(0)), np.sort(c1.dx.sum(0)))
