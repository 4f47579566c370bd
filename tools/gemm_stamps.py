"""Diagnostic: where a chain GEMM launch spends its time, from per-CTA
%globaltimer stamps (GWB_GEMM_TIMING=1, csrc/gemm.cu).  Runs a few
iterations of a BASELINE config on a device-resident session and prints, for
the last GEMM launched, each phase's median / max over the leader CTAs
relative to the first CTA's entry.

    GWB_GEMM_TIMING=1 python tools/gemm_stamps.py c1 [iters]
"""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

os.environ.setdefault("GWB_GEMM_TIMING", "1")
from paper_2205_08115_b200 import abi  # noqa: E402

NAMES = ["entry", "prologue", "pdl_wait", "first_stage", "last_mma", "drained", "stored", "exit"]


def main():
    case = sys.argv[1] if len(sys.argv) > 1 else "c1"
    iters = sys.argv[2] if len(sys.argv) > 2 else "6"
    # prof_session leaves the session's last launch in the stamps buffer; run
    # it in-process so the buffer is still there.
    sys.argv = ["prof_session.py", case, iters]
    import runpy
    runpy.run_path(os.path.join(ROOT, "tools", "prof_session.py"), run_name="__main__")
    lib = abi.load()
    out = (C.c_uint64 * (8 * 1024))()
    cnt = C.c_int32(0)
    lib.gwb_debug_gemm_stamps(out, 1024, C.byref(cnt))
    n = cnt.value
    if n == 0:
        print("no stamps (GWB_GEMM_TIMING unset?)")
        return
    a = np.frombuffer(out, dtype=np.uint64, count=8 * n).reshape(n, 8).astype(np.int64)
    lead = a[0::2]
    t0 = a[:, 0].min()
    rel = (lead - t0) / 1000.0
    print(f"{case}: last GEMM launch, {n} CTAs ({len(lead)} leader CTAs), µs from the first entry")
    for k, name in enumerate(NAMES):
        col = rel[:, k]
        print(f"  {name:12s} min {col.min():8.2f}  median {np.median(col):8.2f}  max {col.max():8.2f}")


if __name__ == "__main__":
    main()
