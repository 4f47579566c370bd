"""Per-iteration split of a device-resident BAPG session (c1 / c2 / c3):
CUDA-graph time per iteration, eager time, and the eager per-half-step
event split between the chain GEMMs and the projection passes.

    python tools/chain_split.py c1
"""
import ctypes as C, os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from harness import instances as I
from paper_2205_08115_b200 import abi
case = sys.argv[1]
inst = {"c1": I.config1, "c2": I.config2, "c3": I.config3}[case]()
n, m = inst.n, inst.m
ldn, ldm = (n + 31) // 32 * 32, (m + 31) // 32 * 32
up = lambda a, ld: torch.nn.functional.pad(torch.tensor(np.ascontiguousarray(a), dtype=torch.float32), (0, ld - a.shape[1])).cuda()
dx, dy = up(inst.dx, ldn), up(inst.dy, ldm)
mu = torch.tensor(inst.mu, dtype=torch.float32).cuda(); nu = torch.tensor(inst.nu, dtype=torch.float32).cuda()
lib = abi.load()
cfg = abi.default_config(rho=inst.solver["rho"], max_iters=2000, rel_tol=1e-30, precision=0)
st = abi.Status(); s = C.c_void_p()
lib.gwb_session_create(C.byref(cfg), n, m, 0, C.byref(s), C.byref(st)); abi.raise_for(st)
lib.gwb_session_load_device(s, dx.data_ptr(), ldn, dy.data_ptr(), ldm, mu.data_ptr(), nu.data_ptr(), None, C.byref(st)); abi.raise_for(st)
lib.gwb_session_reset(s, None, C.byref(st))
L = C.c_int64(0)
lib.gwb_session_iterate(s, 20, None, C.byref(L), C.byref(st))
g, c = C.c_double(), C.c_int64()
lib.gwb_session_kernel_ms(s, 0, C.byref(g), C.byref(c), C.byref(st))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
sp = C.c_void_p(); lib.gwb_session_stream(s, C.byref(sp), C.byref(st)); stream = torch.cuda.ExternalStream(sp.value)
out = {}
for mode in ("graph", "eager"):
    L = C.c_int64(0 if mode == "graph" else -1)
    e0.record(stream)
    lib.gwb_session_iterate(s, 200, None, C.byref(L), C.byref(st))
    e1.record(stream); e1.synchronize()
    out[mode + "_us_per_it"] = e0.elapsed_time(e1) / 200 * 1e3
    out["launches_per_it"] = L.value / 200
lib.gwb_session_kernel_ms(s, 0, C.byref(g), C.byref(c), C.byref(st))
g2, c2 = C.c_double(), C.c_int64()
lib.gwb_session_kernel_ms(s, 1, C.byref(g2), C.byref(c2), C.byref(st))
out.update(chain_us_per_half=g.value * 1e3, proj_us_per_half=g2.value * 1e3, marks=c.value)
print(case, json.dumps(out))
