"""Parity criteria shared by the GPU tests (north_star: final coupling within
1e-4 max-abs relative to its scale, GW objective within 1e-5 relative, the
same argmax node matching).

Argmax ("bit-exact" hard_assignment, tasks.cpp:190-200) is judged row by
row against the reference's 4 largest entries per row (exact fp64 values
and indices, lowest index first on ties):

* the GPU coupling's relative error on those entries, e = max_i,k
  |π[i, idx_k] − v_k| / v_1, is measured exactly (no quantisation);
* decided rows — reference top-2 margin v_1 − v_2 above thr_i = 2.5·e·v_1
  (no error of size e can flip them): the pick must equal the reference's;
* exact fp64 ties (v_1 == v_2): the pick must lie in the tied set;
* the remaining near-ties: the reference's value at the pick must be within
  thr_i of v_1 (a near-tie, never an arbitrary column; a pick outside the
  stored top-4 has reference value ≤ v_4).

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


def top_error(pi: np.ndarray, top_idx: np.ndarray, top_val: np.ndarray) -> float:
    """Max relative (to the row's largest entry) error of `pi` on the
    reference's top-4 entries of every row."""
    got = np.take_along_axis(pi, top_idx.astype(np.int64), axis=1)
    v1 = np.where(top_val[:, :1] > 0, top_val[:, :1], 1.0)
    return float(np.max(np.abs(got - top_val) / v1))


def argmax_check(pick: np.ndarray, pi: np.ndarray, top_idx: np.ndarray, top_val: np.ndarray,
                 min_decided: float, label: str = "", ref_value_at=None,
                 slack: float = 0.0) -> dict:
    """pick: GPU hard_assignment (n); pi: the GPU coupling (n × m);
    ref_value_at(rows, cols) (optional): reference values within ±slack,
    used only for tied rows whose tie set exceeds the stored top-4."""
    pick = np.asarray(pick)
    n = pick.size
    v1, v2, v4 = top_val[:, 0], top_val[:, 1], top_val[:, 3]
    e = top_error(pi, top_idx, top_val)
    thr = 2.5 * max(e, 1e-12) * v1
    tied = v1 == v2
    decided = ~tied & (v1 - v2 > thr)
    in_top = top_idx == pick[:, None]
    known = in_top.any(axis=1)
    ref_at_pick = np.where(known, (top_val * in_top).sum(axis=1), v4)  # ≤ v4 outside top-4
    bad_decided = decided & (pick != top_idx[:, 0])
    bad_tied = tied & known & (ref_at_pick != v1)
    unknown_tied = tied & ~known
    bad_tied |= unknown_tied & (v4 < v1)  # the whole tie set is among the stored top-4
    big = unknown_tied & (v4 == v1)        # tie set of 4 or more: check the full coupling
    if big.any() and ref_value_at is not None:
        rows = np.flatnonzero(big)
        bad_tied[rows] |= ref_value_at(rows, pick[rows]) < v1[rows] - 2 * slack
    near = ~decided & ~tied
    bad_near = near & (ref_at_pick < v1 - thr)
    info = {"rows": n, "decided": int(decided.sum()), "tied": int(tied.sum()),
            "near_ties": int(near.sum()), "top4_rel_err": e,
            "decided_frac": float(decided.mean()), "mismatched_picks": int((pick != top_idx[:, 0]).sum())}
    print(f"argmax {label}: {info}")
    assert not bad_decided.any(), \
        f"{label}: {int(bad_decided.sum())} decided rows differ (first {np.flatnonzero(bad_decided)[:8]})"
    assert not bad_tied.any(), f"{label}: {int(bad_tied.sum())} tied rows picked outside the tied set"
    assert not bad_near.any(), f"{label}: {int(bad_near.sum())} near-tie rows picked a non-maximal column"
    assert decided.mean() >= min_decided, \
        f"{label}: only {decided.mean():.3f} of rows decided (need {min_decided})"
    return info
