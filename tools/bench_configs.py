"""Iterations/s of the BASELINE.json configs c1–c3 (and c4 at reduced n) on
the device-resident session path (CUDA graphs, no host sync), with the
resolved precision.  Diagnostic companion of bench.py (which measures c4)."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2205_08115_b200 import abi
from harness import instances as I

PREC = {"auto": 0, "tf32": 1, "3xtf32": 2, "bf16x3": 3, "bf16x2": 4, "sparse": 5, "fp32": 6, "f16x2": 7}


def session_rate(inst, iters, prec="auto", warm=3):
    lib = abi.load()
    t = lambda a, ld: torch.nn.functional.pad(
        torch.tensor(np.ascontiguousarray(a), dtype=torch.float32), (0, ld - a.shape[1])).cuda()
    ldn = (inst.n + 31) // 32 * 32
    ldm = (inst.m + 31) // 32 * 32
    dx, dy = t(inst.dx, ldn), t(inst.dy, ldm)
    mu = torch.tensor(inst.mu, dtype=torch.float32).cuda()
    nu = torch.tensor(inst.nu, dtype=torch.float32).cuda()
    cfg = abi.default_config(rho=inst.solver["rho"], max_iters=iters + warm + 4, rel_tol=1e-30,
                             precision=PREC[prec])
    st = abi.Status()
    s = C.c_void_p()
    lib.gwb_session_create(C.byref(cfg), inst.n, inst.m, 0, C.byref(s), C.byref(st))
    abi.raise_for(st)
    lib.gwb_session_load_device(s, dx.data_ptr(), ldn, dy.data_ptr(), ldm, mu.data_ptr(),
                                nu.data_ptr(), None, C.byref(st))
    abi.raise_for(st)
    lib.gwb_session_reset(s, None, C.byref(st))
    sp = C.c_void_p()
    lib.gwb_session_stream(s, C.byref(sp), C.byref(st))
    stream = torch.cuda.ExternalStream(sp.value)
    rp, fl = C.c_int32(), C.c_double()
    lib.gwb_session_info(s, C.byref(rp), C.byref(fl), C.byref(st))
    L = C.c_int64(0)
    lib.gwb_session_iterate(s, warm, None, C.byref(L), C.byref(st))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    L = C.c_int64(0)
    lib.gwb_session_iterate(s, iters, None, C.byref(L), C.byref(st))
    e1.record(stream)
    e1.synchronize()
    abi.raise_for(st)
    ms = e0.elapsed_time(e1)
    lib.gwb_session_destroy(s)
    return {"it_per_s": iters / (ms * 1e-3), "ms_per_it": ms / iters,
            "precision": {1: "tf32", 2: "3xtf32", 3: "bf16x3", 4: "bf16x2", 5: "sparse", 6: "fp32", 7: "f16x2", 8: "f16x3"}[rp.value],
            "tflops_alg": fl.value * iters / (ms * 1e-3) / 1e12, "launches": L.value}


if __name__ == "__main__":
    out = {}
    only = None
    for a in sys.argv[1:]:
        if a.startswith("--only="):
            only = a[len("--only="):].split(",")
    cases = [("c1", I.config1, 2000), ("c2", I.config2, 1000), ("c3", I.config3, 500),
             ("c4@8192", lambda: I.config4(n=8192), 20)]
    for name, make, iters in cases:
        if only and name not in only:
            continue
        inst = make()
        out[name] = session_rate(inst, iters)
        print(name, json.dumps(out[name]), flush=True)
        if name in ("c1", "c4@8192") and "--compare" in sys.argv:
            r = session_rate(inst, iters, "bf16x3")
            print(name, "bf16x3", json.dumps(r), flush=True)
