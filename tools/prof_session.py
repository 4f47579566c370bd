"""Drive a few BAPG iterations of one session (device-resident inputs) for
profiling: python tools/prof_session.py [n] [precision] [iters]."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2205_08115_b200 import abi
from harness import instances as I

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
prec = {"auto": 0, "tf32": 1, "3xtf32": 2, "bf16x3": 3, "bf16x2": 4, "sparse": 5, "f16x2": 7}[
    sys.argv[2] if len(sys.argv) > 2 else "auto"]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
e = I.barabasi_albert(n, 5, I.mix_seed(0, 41))
noisy = I.edge_noise(n, e, 0.02, 0.02, I.mix_seed(0, 1))
tgt, _ = I.permute_graph(n, noisy, I.mix_seed(0, 2))
ld = (n + 31) // 32 * 32


def dense(edges):
    d = torch.zeros((n, ld), device="cuda")
    t = torch.from_numpy(edges.astype("int64")).cuda()
    d[t[:, 0], t[:, 1]] = 1.0
    d[t[:, 1], t[:, 0]] = 1.0
    return d


lib = abi.load()
dx, dy = dense(e), dense(tgt)
mu = torch.full((n,), 1.0 / n, device="cuda")
cfg = abi.default_config(rho=0.1, max_iters=iters + 4, rel_tol=1e-30, precision=prec)
st = abi.Status()
s = C.c_void_p()
lib.gwb_session_create(C.byref(cfg), n, n, 0, C.byref(s), C.byref(st))
abi.raise_for(st)
lib.gwb_session_load_device(s, dx.data_ptr(), ld, dy.data_ptr(), ld, mu.data_ptr(), mu.data_ptr(),
                            None, C.byref(st))
abi.raise_for(st)
del dx, dy
lib.gwb_session_reset(s, None, C.byref(st))
L = C.c_int64(0)
lib.gwb_session_iterate(s, iters, None, C.byref(L), C.byref(st))
torch.cuda.synchronize()
abi.raise_for(st)
lib.gwb_session_destroy(s)
print("ok", iters, "iterations, launches", L.value)
