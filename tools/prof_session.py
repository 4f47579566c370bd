"""Drive a few BAPG iterations of one BASELINE config on a device-resident
session (inputs uploaded before, no host sync inside), for ncu:

    python tools/prof_session.py CASE [ITERS] [PRECISION]

CASE: c1 | c2 | c3 | c4 (BA n=20000) | c4@N (BA n=N)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from harness import instances as I  # noqa: E402
from paper_2205_08115_b200 import abi  # noqa: E402

PREC = {"auto": 0, "tf32": 1, "3xtf32": 2, "bf16x3": 3, "bf16x2": 4, "sparse": 5, "fp32": 6,
        "f16x2": 7, "f16x3": 8}
case = sys.argv[1] if len(sys.argv) > 1 else "c4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prec = PREC[sys.argv[3] if len(sys.argv) > 3 else "auto"]
if case.startswith("c4"):
    inst = I.config4(n=int(case[3:]) if "@" in case else 20000)
else:
    inst = {"c1": I.config1, "c2": I.config2, "c3": I.config3}[case]()
n, m = inst.n, inst.m
ldn, ldm = (n + 31) // 32 * 32, (m + 31) // 32 * 32
up = lambda a, ld: torch.nn.functional.pad(
    torch.tensor(np.ascontiguousarray(a), dtype=torch.float32), (0, ld - a.shape[1])).cuda()
dx, dy = up(inst.dx, ldn), up(inst.dy, ldm)
mu = torch.tensor(inst.mu, dtype=torch.float32).cuda()
nu = torch.tensor(inst.nu, dtype=torch.float32).cuda()
lib = abi.load()
cfg = abi.default_config(rho=inst.solver["rho"], max_iters=iters + 4, rel_tol=1e-30, precision=prec)
st = abi.Status()
s = C.c_void_p()
lib.gwb_session_create(C.byref(cfg), n, m, 0, C.byref(s), C.byref(st))
abi.raise_for(st)
lib.gwb_session_load_device(s, dx.data_ptr(), ldn, dy.data_ptr(), ldm, mu.data_ptr(), nu.data_ptr(),
                            None, C.byref(st))
abi.raise_for(st)
del dx, dy
lib.gwb_session_reset(s, None, C.byref(st))
L = C.c_int64(0)
lib.gwb_session_iterate(s, iters, None, C.byref(L), C.byref(st))
torch.cuda.synchronize()
abi.raise_for(st)
rp, fl = C.c_int32(), C.c_double()
lib.gwb_session_info(s, C.byref(rp), C.byref(fl), C.byref(st))
lib.gwb_session_destroy(s)
print("ok", case, iters, "iterations, launches", L.value, "precision", rp.value)
