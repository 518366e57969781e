"""Shared test utilities: bf16-representable inputs, tie-tolerant selection
comparison. Test infrastructure only."""
from __future__ import annotations

import numpy as np


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 to the nearest bf16 (ties to even) and return it as fp32, so
    the identical bytes can be fed to the fp32 oracle and the bf16 pool."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(a.shape)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    return (bf16_round(x).view(np.uint32) >> 16).astype(np.uint16)


def rng_normal(seed: int, shape, scale: float = 1.0) -> np.ndarray:
    g = np.random.default_rng(seed)
    return (g.standard_normal(shape) * scale).astype(np.float32)


ABS_TIE = 1e-30  # criticality below this is numerically zero (< 2^-99 of the total mass H)


def check_selection(ours, ref, crit_ref_full, cand, rel_tol=1e-4, abs_tol=ABS_TIE):
    """Selected sets must be equal except for indices whose reference
    criticality ties the k-th value: |crit - kth| <= rel_tol*|kth| + abs_tol
    (the absolute floor covers fp32-subnormal criticalities,
    which carry no ranking information)."""
    ours = np.asarray(ours, dtype=np.int64)
    ref = np.asarray(ref, dtype=np.int64)
    assert len(ours) == len(ref), (len(ours), len(ref))
    if np.array_equal(ours, ref):
        return 0
    pos = {int(t): i for i, t in enumerate(np.asarray(cand, dtype=np.int64))}
    kth = min(crit_ref_full[pos[int(t)]] for t in ref)
    diff = set(ours.tolist()) ^ set(ref.tolist())
    for t in diff:
        c = crit_ref_full[pos[t]]
        assert abs(c - kth) <= rel_tol * abs(kth) + abs_tol, f"index {t}: crit {c} vs k-th {kth} (not a tie)"
    return len(diff)
