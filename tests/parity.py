"""Parity criteria shared by the GPU tests (north_star: final coupling within
1e-4 max-abs relative to its scale, GW objective within 1e-5 relative, the
same argmax node matching).

Argmax ("bit-exact" hard_assignment, tasks.cpp:190-200) is judged row by
row against the reference coupling:

* decided rows — reference top-2 margin above ``thr`` (a multiple of the
  measured coupling error, so no fp32-level difference can flip them):
  the pick must equal the reference's;
* exact fp64 ties (top-1 == top-2): the pick must lie in the tied set;
* the remaining near-ties: the pick's reference value must be within
  ``thr`` of the row maximum (a near-tie, never an arbitrary column).

Each case asserts a minimum decided fraction and reports the undecided
count, so the check cannot pass vacuously.
"""
from __future__ import annotations

import numpy as np

PI_TOL = 1e-4
OBJ_TOL = 1e-5
QUANT = 0.5 / 65535.0  # fingerprint quantisation (fraction of scale)


def dequantise(q: np.ndarray, scale: float) -> np.ndarray:
    return q.astype(np.float64) * (scale / 65535.0)


def argmax_check(pick: np.ndarray, ref_value_at, top_idx: np.ndarray, top_val: np.ndarray,
                 scale: float, thr: float, min_decided: float, label: str = "") -> dict:
    """pick: GPU hard_assignment (n); ref_value_at(rows, cols) -> reference
    values (exact or dequantised, within ``slack``); top_idx / top_val: the
    reference's 4 largest per row (fp64, lowest index first on ties)."""
    pick = np.asarray(pick)
    n = pick.size
    v1, v2 = top_val[:, 0], top_val[:, 1]
    margin = (v1 - v2) / scale
    tied = v1 == v2
    decided = margin > thr
    rows = np.arange(n)
    bad_decided = decided & (pick != top_idx[:, 0])
    # Value of the reference coupling at the GPU's pick: exact when the pick
    # is one of the stored top-4 entries, else from ref_value_at.
    at = ref_value_at(rows, pick)
    in_top = top_idx == pick[:, None]
    exact = np.where(in_top.any(axis=1), (top_val * in_top).sum(axis=1), at)
    exact_known = in_top.any(axis=1)
    bad_tied = tied & exact_known & (exact != v1)
    bad_tied |= tied & ~exact_known & (at < v1 - 2 * QUANT * scale)
    undecided = ~decided & ~tied
    bad_near = undecided & (exact < v1 - thr * scale - 2 * QUANT * scale)
    info = {"rows": n, "decided": int(decided.sum()), "tied": int(tied.sum()),
            "near_ties": int(undecided.sum()), "threshold": thr,
            "decided_frac": float(decided.mean())}
    print(f"argmax {label}: {info}")
    assert not bad_decided.any(), \
        f"{label}: {int(bad_decided.sum())} decided rows differ (first {np.flatnonzero(bad_decided)[:8]})"
    assert not bad_tied.any(), f"{label}: {int(bad_tied.sum())} tied rows picked outside the tied set"
    assert not bad_near.any(), f"{label}: {int(bad_near.sum())} near-tie rows picked a non-maximal column"
    assert decided.mean() >= min_decided, \
        f"{label}: only {decided.mean():.3f} of rows decided (need {min_decided})"
    return info


def decided_threshold(err: float) -> float:
    """Rows with a reference margin above 2.5x the measured max coupling
    error (fraction of scale) cannot flip."""
    return 2.5 * max(err, 1e-9)
