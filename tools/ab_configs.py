"""A/B timing of the small configs on device-resident sessions (CUDA graphs):
python tools/ab_configs.py c1 c2 c3 — run it under different GWB_* knobs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from harness import instances as I  # noqa: E402
from paper_2205_08115_b200 import abi  # noqa: E402

iters = {"c1": 2000, "c2": 1000, "c3": 500}
make = {"c1": I.config1, "c2": I.config2, "c3": I.config3}
lib = abi.load()
knobs = {k: v for k, v in os.environ.items() if k.startswith("GWB_")}
for c in sys.argv[1:]:
    inst = make[c]()
    r = bench.session_run(lib, abi, torch, inst, iters[c], 0)
    print(c, knobs, f"{iters[c] / (r['ms'] * 1e-3):.1f} it/s", f"{r['ms'] / iters[c] * 1e3:.1f} us/it",
          "launches", r["launches"], flush=True)
