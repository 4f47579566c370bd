"""CPU checks of the full-size reference fingerprints (tests/golden/fp_*.npz,
tools/make_fingerprints.py): the harness regenerates the same inputs (SHA-256),
the fingerprints are internally consistent, and the C restatement of the
oracle reproduces the reference's fingerprint on the configs it finishes in
seconds (c3 with and without the jittered start)."""
import glob
import os

import numpy as np
import pytest

from harness import cases as C
from harness import instances as I
from paper_2205_08115_b200 import abi
from tests.parity import QUANT, dequantise

HERE = os.path.join(os.path.dirname(__file__), "golden")
FPS = sorted(glob.glob(os.path.join(HERE, "fp_*.npz")))
SMALL = ["c1", "c1_jit", "c3", "c3_jit", "c2", "c4_ba4000", "c4_ba4000_jit", "c4_hbpg_ba4000"]


def have(name):
    return os.path.exists(os.path.join(HERE, f"fp_{name}.npz"))


def test_fingerprints_present():
    names = {os.path.basename(p)[3:-4] for p in FPS}
    assert {"c1", "c1_jit", "c3", "c3_jit"} <= names, names


@pytest.mark.parametrize("name", SMALL)
def test_inputs_regenerate(name):
    if not have(name):
        pytest.skip("fingerprint not generated yet")
    z = np.load(os.path.join(HERE, f"fp_{name}.npz"))
    inst, init = C.CASES[name][0]()
    assert C.sha(inst.dx, inst.dy, inst.mu, inst.nu, init) == str(z["input_sha"])
    # Internal consistency: the quantised coupling, top-4 and sums agree.
    scale = float(z["scale"])
    pi = dequantise(z["q"], scale)
    assert np.abs(pi.max(axis=1) - z["top_val"][:, 0]).max() <= QUANT * scale * 1.01
    assert np.abs(pi.sum(axis=1) - z["rowsum"]).max() <= QUANT * scale * pi.shape[1]


def test_c5_inputs_regenerate():
    if not have("c5"):
        pytest.skip("fingerprint not generated yet")
    z = np.load(os.path.join(HERE, "fp_c5.npz"))
    for k in (0, 1, int(z["count"]) - 1):
        i = I.config5_problem(k)
        assert C.sha(i.dx, i.dy, i.mu, i.nu, None) == str(z["input_sha"][k])


@pytest.mark.parametrize("name", ["c3", "c3_jit"])
def test_port_reproduces_reference_fingerprint(port, name):
    """The C restatement follows the reference's full-size c3 trace record by
    record (the first 60 of its 500 iterations: the port's cost here is
    minutes per 500)."""
    z = np.load(os.path.join(HERE, f"fp_{name}.npz"))
    make, over, _ = C.CASES[name]
    inst, init = make()
    kw = dict(inst.solver)
    kw.update(over, quiet=1, max_iters=60)
    cfg = abi.default_config(**kw)
    r = port.solve(cfg, inst.dx, inst.dy, inst.mu, inst.nu, initial=init)
    assert r.code == 0, r.message
    assert r.iterations_used == 60
    np.testing.assert_allclose([t["objective"] for t in r.trace], z["trace"][:60, 1], rtol=1e-9)
    np.testing.assert_allclose([t["rel_change"] for t in r.trace], z["trace"][:60, 4], rtol=1e-6)
