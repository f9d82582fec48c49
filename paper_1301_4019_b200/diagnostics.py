"""Weight validation and the log-weight adapter on the GPU.

Mirrors the two hot-path functions of pfresample.diagnostics:
check_weights (diagnostics.py:38-51) and logweights_to_weights (138-155).
The analysis helpers of that module (ESS, MSE, synthetic weight sets) are not
part of the resampling step; ``ess`` is provided as a device reduction because
the particle filter driver decides on it.
"""

from __future__ import annotations

import torch

from . import _lib as L

__all__ = ["check_weights", "logweights_to_weights", "ess", "resampling_mse"]


def check_weights(w, require_positive_total: bool = True, name: str = "w") -> torch.Tensor:
    """Validate: 1-D, finite, non-negative, not all zero (diagnostics.py:38-51).
    Returns the device tensor (float input kept, other input cast to float64)."""
    w = L.as_weights(w, name)
    st = L.new_status()
    L.call("pfr_check_weights", w.data_ptr(), w.numel(), L.dtype_code(w), st.data_ptr(), L.stream_handle())
    L.raise_weight_errors(L.read_status(st), name, require_positive_total)
    return w


def logweights_to_weights(lw) -> torch.Tensor:
    """w = exp(lw - max lw); -inf -> 0; NaN/+inf or all -inf rejected
    (diagnostics.py:138-155)."""
    lw = L.as_weights(lw, "log-weight vector")
    w = torch.empty_like(lw)
    st = L.new_status()
    ws, wsb = L.workspace(lw.numel())
    L.call("pfr_logweights_to_weights", lw.data_ptr(), w.data_ptr(), lw.numel(), L.dtype_code(lw), st.data_ptr(),
           ws, wsb, L.stream_handle())
    bits = L.read_status(st)
    if bits & L.ST_NONFINITE:
        raise ValueError("log-weights may not contain NaN or +inf")
    if not bits & L.ST_POSITIVE:
        raise ValueError("all log-weights are -inf: no positive weight")
    return w


def _weight_stats(w, o=None):
    out = torch.empty(4, dtype=torch.float64, device=w.device)
    ws, wsb = L.workspace(w.numel())
    L.call("pfr_weight_stats", w.data_ptr(), w.numel(), L.dtype_code(w), L.ptr(o),
           L.dtype_code(o) if o is not None else L.I32, out.data_ptr(), ws, wsb, L.stream_handle())
    return out.cpu().numpy()


def ess(w) -> float:
    """Effective sample size (sum w)^2 / (w . w) (diagnostics.py:54-63): one
    deterministic device pass (pfr_weight_stats)."""
    w = check_weights(w)
    return float(_weight_stats(w)[2])


def resampling_mse(o, w) -> float:
    """(1/N) sum_i (o[i]/N - w[i]/sum w)^2 in float64 (diagnostics.py:66-80),
    fused with the weight sums in one device pass."""
    w = check_weights(w)
    o = L.as_index(o, "offspring vector")
    if o.numel() != w.numel():
        raise ValueError(f"offspring and weight vectors differ in length: ({o.numel()},) vs ({w.numel()},)")
    return float(_weight_stats(w, o)[3])
