"""GPU prefix sums, adjacent difference, totals and binary search.

Mirrors pfresample.primitives (primitives.py:34-106) over device tensors.
All floating-point scans run through the single-pass deterministic
lookback-tree kernel (csrc/pfr_scan.cu): the association differs from
np.cumsum's serial fold (results agree to rounding), but it is fixed, so
every run and every launch geometry returns the same bits.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L

__all__ = [
    "stable_sum",
    "inclusive_prefix_sum",
    "exclusive_prefix_sum",
    "adjacent_difference",
    "vector_sum",
    "lower_bound",
]


def _scan(w, exclusive: bool, accum=None, monotone: bool = False, name: str = "w"):
    w = L.as_weights(w, name)
    n = w.numel()
    out = torch.empty_like(w)
    total = torch.empty(1, dtype=torch.float64, device=w.device)
    st = L.new_status()
    ws, wsb = L.workspace(n)
    flags = L.accum_code(accum) | (L.SCAN_MONOTONE if monotone else 0)
    dt = L.dtype_code(w)
    L.call("pfr_scan", w.data_ptr(), out.data_ptr(), n, dt, dt, flags, int(exclusive), total.data_ptr(),
           st.data_ptr(), ws, wsb, L.stream_handle())
    if L.config.check:
        bits = L.read_status(st)
        if bits & L.ST_NONFINITE:
            raise ValueError(f"{name} must be finite (no NaN or infinity)")
    return out, total


def inclusive_prefix_sum(w, *, accum=None, monotone: bool = False) -> torch.Tensor:
    """result[i] = w[0] + ... + w[i] in the input precision (primitives.py:34-42).

    ``accum="f64"`` (default) carries float32 inputs in float64 and rounds
    once on output; ``accum="native"`` accumulates in float32 with the
    parallel (tree) association; ``accum="serial"`` performs the reference's
    own left-to-right fold in the input dtype, so the result equals
    ``np.cumsum`` bit for bit (parity mode, one serial GPU thread).
    ``monotone=True`` (for non-negative inputs) repairs ulp-level
    non-monotonicity with an exact running max."""
    return _scan(w, False, accum, monotone)[0]


def exclusive_prefix_sum(w, *, accum=None, monotone: bool = False) -> torch.Tensor:
    """result[0] = 0, result[i] = inclusive[i-1] exactly (primitives.py:45-51)."""
    return _scan(w, True, accum, monotone)[0]


def vector_sum(w, *, accum=None) -> torch.Tensor:
    """Total, bit-identical to inclusive_prefix_sum(w)[-1] (primitives.py:60-66)."""
    out, _ = _scan(w, False, accum)
    return out[-1]


def adjacent_difference(W) -> torch.Tensor:
    """result[0] = W[0], result[i] = W[i] - W[i-1] (primitives.py:54-57)."""
    W = L.as_weights(W, "W")
    out = torch.empty_like(W)
    st = L.new_status()
    dt = L.dtype_code(W)
    L.call("pfr_adjacent_difference", W.data_ptr(), out.data_ptr(), W.numel(), dt, dt, st.data_ptr(),
           L.stream_handle())
    if L.config.check and L.read_status(st) & L.ST_NONFINITE:
        raise ValueError("W must be finite (no NaN or infinity)")
    return out


def lower_bound(W, u, *, index_dtype=None):
    """Smallest j with W[j] >= u, clamped to N-1 (primitives.py:91-106).
    Comparisons are made in float64, as numpy promotes float32 W."""
    W = L.as_weights(W, "W")
    scalar = not isinstance(u, torch.Tensor) and torch.tensor(u).dim() == 0
    ut = torch.as_tensor(u, dtype=torch.float64).reshape(-1).to(W.device).contiguous()
    out = torch.empty(ut.numel(), dtype=torch.int32, device=W.device)
    L.call("pfr_lower_bound", W.data_ptr(), W.numel(), L.dtype_code(W), ut.data_ptr(), ut.numel(), out.data_ptr(),
           L.stream_handle())
    out = L.to_index_dtype(out, index_dtype)
    return out[0] if scalar else out


def stable_sum(w):
    """Balanced pairwise-tree sum of the zero-padded power-of-two vector
    (primitives.py:69-88), bit-identical to the reference; returns a numpy
    scalar of the input dtype."""
    w = L.as_weights(w, "vector")
    out = torch.empty(1, dtype=torch.float64, device=w.device)
    ws, wsb = L.workspace(w.numel())
    st = L.new_status()
    L.call("pfr_check_weights", w.data_ptr(), w.numel(), L.dtype_code(w), st.data_ptr(), L.stream_handle())
    L.call("pfr_stable_sum", w.data_ptr(), w.numel(), L.dtype_code(w), out.data_ptr(), ws, wsb, L.stream_handle())
    if L.read_status(st) & L.ST_NONFINITE:
        raise ValueError("vector must be finite (no NaN or infinity)")
    t = np.float32 if w.dtype == torch.float32 else np.float64
    return t(float(out.item()))
