"""write_coupling_csv throughput: device formatting (csrc/csv.cu) through
gwb_write_coupling_csv_file to /dev/null (host fp64 input: includes the
H2D copy and the text D2H), against the oracle's "%.17g" loop (one core)
on a sample.  One JSON line per size."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_08115_b200 as gw  # noqa: E402
from oracle.bindings import Oracle  # noqa: E402


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [2048, 8192]
    port = Oracle("port")
    for n in sizes:
        rng = np.random.default_rng(n)
        a = np.asfortranarray(rng.random((n, n)) / (n * n))
        gw.write_coupling_csv_file("/dev/null", a[:64, :64])  # warm-up
        t = time.perf_counter()
        gw.write_coupling_csv_file("/dev/null", a)
        dt = time.perf_counter() - t
        nbytes = len(gw.format_coupling_csv(a[:256, :256])) * (n / 256) ** 2
        s = min(n, 1024)
        t = time.perf_counter()
        port.format_coupling_csv(np.asfortranarray(a[:s, :s]))
        ct = time.perf_counter() - t
        print(json.dumps(dict(n=n, entries=n * n, seconds=round(dt, 4),
                              entries_per_s=round(n * n / dt), text_gb_per_s=round(nbytes / dt / 1e9, 2),
                              cpu_entries_per_s=round(s * s / ct), cpu_sample=f"{s}x{s}, 1 core",
                              speedup=round((n * n / dt) / (s * s / ct), 1))), flush=True)


if __name__ == "__main__":
    main()
