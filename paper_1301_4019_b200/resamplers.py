"""The five resamplers on the GPU, plus the reference's facade.

Mirrors pfresample.resamplers (resamplers.py:56-397): same names, arguments,
keyword hooks (``uniforms=``, ``offset=``, ``return_trips=``) and errors.
Weights stay on the device; outputs are device tensors.

Randomness: ``rng`` is an RngStream (this package's or the reference's).  With
``rng_mode="numpy"`` the kernels replay numpy's Philox4x64-10 stream exactly
as the reference consumes it, so results match the reference bit for bit
(up to rounding-fragile positions of the float scan); with the default
``rng_mode="philox"`` they use the GPU's own Philox4x32-10 counters, which
is faster and statistically equivalent.

``deliver`` is the bench's timed region (bench.py:155-161): resample, expand
and permute to an in-place-valid ancestry.  For systematic/stratified it runs
the fused offspring -> permute path that never materialises the sorted
ancestry.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .ancestry import cumulative_offspring_to_ancestors, permute_parallel
from .rng import as_stream

__all__ = [
    "ALGORITHMS",
    "ResamplerConfig",
    "ResampleOutput",
    "multinomial_ancestors",
    "multinomial_ancestors_serial",
    "stratified_cumulative_offspring",
    "systematic_cumulative_offspring",
    "stratum_offset_kernel",
    "metropolis_num_steps",
    "metropolis_ancestors",
    "rejection_ancestors",
    "rejection_ancestors_capped",
    "resolve_metropolis_steps",
    "resample_ancestors",
    "deliver",
]

MAX_REJECTION_ROUNDS = 100_000  # resamplers.py:45

# purpose tags of the own-stream counters (csrc/pfr_rng.cuh)
_TAG_SYSTEMATIC = 0x5359

_ANCESTRY = ("multinomial", "multinomial-serial", "metropolis", "rejection", "rejection-capped")
_OFFSPRING = ("stratified", "systematic")
ALGORITHMS = _ANCESTRY[:2] + _OFFSPRING + _ANCESTRY[2:]


@dataclass(frozen=True)
class ResamplerConfig:
    """Algorithm selector and its parameters (resamplers.py:318-338)."""

    algorithm: str = "systematic"
    b: int | None = None
    p_star: float | None = None
    epsilon: float | None = None
    sup_w: float | None = None
    sup_v: float | None = None

    def __post_init__(self):
        if self.algorithm not in ALGORITHMS:
            raise ValueError(f"unknown algorithm {self.algorithm!r}; choose from {ALGORITHMS}")


@dataclass(frozen=True)
class ResampleOutput:
    """Ancestry plus optional carried weights and per-algorithm extras (resamplers.py:341-347)."""

    ancestors: torch.Tensor
    weights: torch.Tensor | None = None
    extras: dict | None = None


# ---------------------------------------------------------------------------
# helpers


def _rng(rng, mode=None, arrays=False) -> L.PfrRng:
    k0, k1 = as_stream(rng).key() if rng is not None else (0, 0)
    code = L.RNG_ARRAYS if arrays else L.rng_mode_code(mode)
    return L.PfrRng(k0, k1, code, 0)


def _weights_checked(w, require_positive_total=True):
    """Enqueue the validation pass; returns (device tensor, status)."""
    w = L.as_weights(w)
    st = L.new_status()
    L.call("pfr_check_weights", w.data_ptr(), w.numel(), L.dtype_code(w), st.data_ptr(), L.stream_handle())
    return w, st


def _raise(st, require_positive_total=True, extra=None):
    if not L.config.check:
        return
    bits = L.read_status(st)
    L.raise_weight_errors(bits, "w", require_positive_total)
    if extra:
        extra(bits)


def _systematic_offset(rng, mode) -> float:
    r = _rng(rng, mode)
    return float(L.lib().pfr_stream_uniform(r, 0, _TAG_SYSTEMATIC))


# ---------------------------------------------------------------------------
# offspring algorithms (cumulative offspring vectors)


def systematic_cumulative_offspring(w, rng, *, offset=None, rng_mode=None, accum=None, index_dtype=None):
    """Systematic resampling: one shared offset (resamplers.py:127-136).
    O[i] = min(N, floor(N W[i]/W[N-1] + u)); fused scan + offspring kernels."""
    w = L.as_weights(w)
    u = _systematic_offset(rng, rng_mode) if offset is None else float(offset)
    n = w.numel()
    O = torch.empty(n, dtype=torch.int32, device=w.device)
    st = L.new_status()
    ws, wsb = L.workspace(n)
    L.call("pfr_cumulative_offspring", w.data_ptr(), n, L.dtype_code(w), L.accum_code(accum), 0, u, None, None,
           O.data_ptr(), st.data_ptr(), ws, wsb, L.stream_handle())
    _raise(st)
    return L.to_index_dtype(O, index_dtype)


def stratified_cumulative_offspring(w, rng, *, uniforms=None, rng_mode=None, accum=None, index_dtype=None):
    """Stratified resampling: one offset per stratum (resamplers.py:105-124).
    Offsets come from ``uniforms`` (float64, cast to the weight dtype) or are
    evaluated on the fly from the stream: no offset array in HBM."""
    w = L.as_weights(w)
    n = w.numel()
    O = torch.empty(n, dtype=torch.int32, device=w.device)
    uni = None
    if uniforms is not None:
        uni = torch.as_tensor(np.asarray(uniforms, dtype=np.float64) if not isinstance(uniforms, torch.Tensor)
                              else uniforms, dtype=torch.float64).to(w.device).contiguous()
        if uni.numel() != n:
            raise ValueError("need one uniform per stratum")
    r = _rng(rng, rng_mode)
    st = L.new_status()
    ws, wsb = L.workspace(n)
    L.call("pfr_cumulative_offspring", w.data_ptr(), n, L.dtype_code(w), L.accum_code(accum), 1, 0.0, L.ptr(uni),
           r, O.data_ptr(), st.data_ptr(), ws, wsb, L.stream_handle())
    _raise(st)
    return L.to_index_dtype(O, index_dtype)


def stratum_offset_kernel(r: float, u: float, n: int, dtype=np.float64) -> int:
    """Scalar min(N, floor(r + u)) in a chosen precision (resamplers.py:156-165);
    the device kernels use the same expression per element."""
    t = np.dtype(dtype).type
    return int(min(n, math.floor(float(t(r) + t(u)))))


# ---------------------------------------------------------------------------
# ancestry algorithms


def multinomial_ancestors(w, rng, *, uniforms=None, rng_mode=None, accum=None, index_dtype=None):
    """N independent categorical draws (resamplers.py:56-74).

    ``uniforms``: pre-scaled draws in [0, W[N-1]) -> binary search (parity);
    numpy mode: the reference's draws replayed -> binary search (parity);
    philox mode: sorted order statistics from exponential spacings, searched
    in W -> a sorted ancestry (the same multinomial law).  The weight scan
    inside pfr_multinomial reports check_weights' flags (no separate pass)."""
    w = L.as_weights(w)
    st = L.new_status()
    n = w.numel()
    a = torch.empty(n, dtype=torch.int32, device=w.device)
    uni = None
    if uniforms is not None:
        uni = torch.as_tensor(uniforms, dtype=torch.float64).reshape(-1).to(w.device).contiguous()
    r = _rng(rng, rng_mode)
    ws, wsb = L.workspace(n)
    L.call("pfr_multinomial", w.data_ptr(), n, L.dtype_code(w), L.accum_code(accum), r, L.ptr(uni), 0,
           a.data_ptr(), st.data_ptr(), ws, wsb, L.stream_handle())
    _raise(st)
    return L.to_index_dtype(a, index_dtype)


def multinomial_ancestors_serial(w, rng, *, rng_mode=None, accum=None, index_dtype=None):
    """Sorted multinomial via order statistics (resamplers.py:77-102).
    numpy mode replays Code 4's log-spacing construction with the reference's
    draws (a parallel scan of ln(d)/(i+1)); philox mode uses exponential
    spacings.  Output is sorted."""
    w, st = _weights_checked(w)
    n = w.numel()
    a = torch.empty(n, dtype=torch.int32, device=w.device)
    mode = L.rng_mode_code(rng_mode)
    r = _rng(rng, rng_mode)
    ws, wsb = L.workspace(n)
    L.call("pfr_multinomial", w.data_ptr(), n, L.dtype_code(w), L.accum_code(accum), r, None,
           1 if mode == L.RNG_NUMPY else 0, a.data_ptr(), st.data_ptr(), ws, wsb, L.stream_handle())
    _raise(st)
    return L.to_index_dtype(a, index_dtype)


def metropolis_num_steps(p_star: float, epsilon: float | None, n: int) -> int:
    """Smallest B with lambda^B max(alpha, beta)/(alpha+beta) < epsilon for the
    two-state occupancy model (resamplers.py:168-201)."""
    if not 0.0 < p_star <= 1.0:
        raise ValueError("p_star must lie in (0, 1]")
    eps = p_star * 1e-2 if epsilon is None else epsilon
    if not 0.0 < eps < p_star:
        raise ValueError("epsilon must lie in (0, p_star)")
    if n < 2:
        raise ValueError("need at least 2 particles")
    alpha = (1.0 - p_star) / (n * p_star)
    beta = 1.0 / n
    lam = 1.0 - alpha - beta
    if lam <= 0.0:
        raise ValueError(
            f"bias bound invalid: 1 - alpha - beta = {lam} <= 0 (p_star={p_star} too small relative to N={n})")
    bound = math.log(eps * (alpha + beta) / max(alpha, beta)) / math.log(lam)
    return max(1, math.floor(bound) + 1)


def metropolis_ancestors(w, b: int, rng, *, u_draws=None, j_draws=None, rng_mode=None, index_dtype=None,
                         _positive: bool = False):
    """N independent B-step Metropolis chains (resamplers.py:204-234).
    ``u_draws``/``j_draws`` (shape (B, N)) replay supplied draws (any N);
    numpy mode replays the reference stream (power-of-two N).  In philox mode
    the kernel validates w itself as each chain reads its own weight."""
    own = u_draws is None and j_draws is None and (rng_mode or L.config.rng_mode) == "philox"
    if own:
        w = L.as_weights(w)
        st = L.new_status()
    else:
        w, st = _weights_checked(w, require_positive_total=False)
    b = int(b)
    if b < 0:
        raise ValueError("number of chain steps must be non-negative")
    n = w.numel()
    a = torch.empty(n, dtype=torch.int32, device=w.device)
    ud = jd = None
    if u_draws is not None or j_draws is not None:
        ud = torch.as_tensor(u_draws, dtype=torch.float64).to(w.device).contiguous().reshape(-1)
        jd = torch.as_tensor(j_draws).to(w.device).to(torch.int64).contiguous().reshape(-1)
        if ud.numel() != b * n or jd.numel() != b * n:
            raise ValueError("u_draws and j_draws must have shape (B, N)")
        r = _rng(None, arrays=True)
    else:
        r = _rng(rng, rng_mode)
    L.call("pfr_metropolis", w.data_ptr(), n, L.dtype_code(w), b, r, L.ptr(ud), L.ptr(jd), L.I64, a.data_ptr(),
           st.data_ptr(), None, 0, L.stream_handle())

    def extra(bits):
        if bits & L.ST_RANGE:
            raise ValueError("proposal indices must lie in [0, N)")

    _raise(st, require_positive_total=_positive, extra=extra)
    return L.to_index_dtype(a, index_dtype)


def _rejection(w, bound, cap, rng, rng_mode, max_rounds, return_trips, index_dtype, positive=False):
    bound = float(bound)
    if not math.isfinite(bound) or bound <= 0:
        raise ValueError(f"weight bound must be finite and positive, got {bound}")
    w = L.as_weights(w)
    st = L.new_status()  # pfr_rejection reports check_weights' flags (the certain-reject table pass)
    n = w.numel()
    a = torch.empty(n, dtype=torch.int32, device=w.device)
    trips = torch.empty(n, dtype=torch.int32, device=w.device) if return_trips else None
    out_w = torch.empty_like(w) if cap else None
    r = _rng(rng, rng_mode)
    ws, wsb = L.workspace(n)
    L.call("pfr_rejection", w.data_ptr(), n, L.dtype_code(w), bound if not cap else 0.0, bound if cap else 0.0, r,
           int(max_rounds), a.data_ptr(), L.ptr(trips), L.ptr(out_w), st.data_ptr(), ws, wsb, L.stream_handle())

    def extra(bits):
        if bits & L.ST_NOPROGRESS:
            raise RuntimeError(f"rejection resampling made no progress after {max_rounds} rounds; "
                               f"weight bound {bound} is far above every weight")

    _raise(st, require_positive_total=positive, extra=extra)
    a = L.to_index_dtype(a, index_dtype)
    return a, trips, out_w


def rejection_ancestors(w, sup_w: float, rng, *, return_trips: bool = False, rng_mode=None,
                        max_rounds: int = MAX_REJECTION_ROUNDS, index_dtype=None, _positive: bool = False):
    """Rejection with a first deterministic self-proposal (resamplers.py:237-255).

    philox mode: persistent warps with lane refill, each slot on its own
    counter-based stream; numpy mode: the reference's round-synchronous loop
    (resamplers.py:282-310) replayed on its own draws -- same ancestry and
    trip counts bit for bit (csrc/pfr_rejreplay.cu)."""
    a, trips, _ = _rejection(w, sup_w, False, rng, rng_mode, max_rounds, return_trips, index_dtype, _positive)
    return (a, trips.to(torch.int64)) if return_trips else a


def rejection_ancestors_capped(w, sup_v: float, rng, *, return_trips: bool = False, rng_mode=None,
                               max_rounds: int = MAX_REJECTION_ROUNDS, index_dtype=None, _positive: bool = False):
    """Rejection against min(w, sup_v) with importance weights w[a]/v[a]
    (resamplers.py:258-279)."""
    a, trips, out_w = _rejection(w, sup_v, True, rng, rng_mode, max_rounds, return_trips, index_dtype, _positive)
    return (a, out_w, trips.to(torch.int64)) if return_trips else (a, out_w)


# ---------------------------------------------------------------------------
# facade


def resolve_metropolis_steps(w, config: ResamplerConfig) -> int:
    """B from the config or the two-state recipe (resamplers.py:350-359)."""
    if config.b is not None:
        return int(config.b)
    p_star = config.p_star
    if p_star is None:
        wt = L.as_weights(w)
        total = float(wt.sum(dtype=torch.float64))
        if total <= 0:
            raise ValueError("cannot derive p_star from an all-zero weight vector")
        p_star = min(1.0, float(wt.max()) / total)
    return metropolis_num_steps(p_star, config.epsilon, L.as_weights(w).numel())


def resample_ancestors(w, config: ResamplerConfig, rng, **kw) -> ResampleOutput:
    """Run the configured resampler and return the (unpermuted) ancestry
    (resamplers.py:362-397)."""
    w = L.as_weights(w)
    alg = config.algorithm
    if alg == "multinomial":
        return ResampleOutput(multinomial_ancestors(w, rng, **kw), extras={})
    if alg == "multinomial-serial":
        return ResampleOutput(multinomial_ancestors_serial(w, rng, **kw), extras={})
    if alg == "stratified":
        O = stratified_cumulative_offspring(w, rng, **kw)
        return ResampleOutput(cumulative_offspring_to_ancestors(O), extras={})
    if alg == "systematic":
        O = systematic_cumulative_offspring(w, rng, **kw)
        return ResampleOutput(cumulative_offspring_to_ancestors(O), extras={})
    kw.pop("accum", None)
    # check_weights(w) with a positive total up front (resamplers.py:372): the
    # ancestry kernels report the flags, raised here with the facade's rule
    kw["_positive"] = True
    if alg == "metropolis":
        b = resolve_metropolis_steps(w, config)
        return ResampleOutput(metropolis_ancestors(w, b, rng, **kw), extras={"B": b})
    if alg == "rejection":
        sup = config.sup_w if config.sup_w is not None else float(w.max())
        a, trips = rejection_ancestors(w, sup, rng, return_trips=True, **kw)
        return ResampleOutput(a, extras={"mean_trips": float(trips.double().mean())})
    if alg == "rejection-capped":
        if config.sup_v is None:
            raise ValueError("rejection-capped requires sup_v")
        a, out_w, trips = rejection_ancestors_capped(w, config.sup_v, rng, return_trips=True, **kw)
        return ResampleOutput(a, weights=out_w, extras={"mean_trips": float(trips.double().mean())})
    raise ValueError(f"unknown algorithm {alg!r}")


def deliver(w, config: ResamplerConfig, rng, *, rng_mode=None, accum=None, index_dtype=None,
            return_max_steps: bool = False, out: torch.Tensor | None = None, log_weights: bool = False):
    """Resample and permute to an in-place-valid ancestry c (o[i] > 0 => c[i] = i):
    the bench's delivery contract (bench.py:155-161).  Equals
    permute_parallel(resample_ancestors(w, config, rng).ancestors).

    ``log_weights=True``: ``w`` holds log-weights; equals the same call on
    ``logweights_to_weights(w)`` (diagnostics.py:138-155).  For systematic /
    stratified the conversion is fused into the delivery (w is never stored)."""
    alg = config.algorithm
    if log_weights and alg not in _OFFSPRING:
        from .diagnostics import logweights_to_weights

        w = logweights_to_weights(w)
        log_weights = False
    if alg in _OFFSPRING:
        w = L.as_weights(w)
        n = w.numel()
        c = out if out is not None else torch.empty(n, dtype=torch.int32, device=w.device)
        steps = torch.zeros(1, dtype=torch.int32, device=w.device) if return_max_steps else None
        st = L.new_status()
        ws, wsb = L.workspace(n)
        strat = alg == "stratified"
        u = 0.0 if strat else _systematic_offset(rng, rng_mode)
        r = _rng(rng, rng_mode)
        entry = "pfr_deliver_offspring_logw" if log_weights else "pfr_deliver_offspring"
        L.call(entry, w.data_ptr(), n, L.dtype_code(w), L.accum_code(accum), int(strat), u, None,
               r, c.data_ptr(), None, L.ptr(steps), st.data_ptr(), ws, wsb, L.stream_handle())
        if log_weights and L.config.check:
            bits = L.read_status(st)
            if bits & L.ST_NONFINITE:
                raise ValueError("log-weights may not contain NaN or +inf")
            if not bits & L.ST_POSITIVE:
                raise ValueError("all log-weights are -inf: no positive weight")
        else:
            _raise(st)
        c = L.to_index_dtype(c, index_dtype) if out is None else c
        return (c, int(steps.item())) if return_max_steps else c
    if alg == "metropolis" and (rng_mode or L.config.rng_mode) == "philox":
        # fused: the chains make the permute's claims as they finish
        w = L.as_weights(w)
        b = resolve_metropolis_steps(w, config)
        n = w.numel()
        c = out if out is not None else torch.empty(n, dtype=torch.int32, device=w.device)
        steps = torch.zeros(1, dtype=torch.int32, device=w.device) if return_max_steps else None
        st = L.new_status()
        ws, wsb = L.workspace(n)
        L.call("pfr_deliver_metropolis", w.data_ptr(), n, L.dtype_code(w), int(b), _rng(rng, rng_mode),
               c.data_ptr(), L.ptr(steps), st.data_ptr(), ws, wsb, L.stream_handle())
        _raise(st, require_positive_total=True)  # resample_ancestors' check_weights (resamplers.py:372)
        c = L.to_index_dtype(c, index_dtype) if out is None else c
        return (c, int(steps.item())) if return_max_steps else c
    if alg in ("rejection", "multinomial") and (rng_mode or L.config.rng_mode) == "philox":
        # fused: the resampler makes the permute's claims as it writes each slot
        # the resamplers report check_weights' flags themselves (the rejection
        # table pass, the multinomial weight scan)
        w = L.as_weights(w)
        st = L.new_status()
        n = w.numel()
        c = out if out is not None else torch.empty(n, dtype=torch.int32, device=w.device)
        steps = torch.zeros(1, dtype=torch.int32, device=w.device) if return_max_steps else None
        ws, wsb = L.workspace(n)
        r = _rng(rng, rng_mode)
        extra = None
        if alg == "rejection":
            bound = float(config.sup_w) if config.sup_w is not None else float(w.max())
            if not math.isfinite(bound) or bound <= 0:
                raise ValueError(f"weight bound must be finite and positive, got {bound}")
            L.call("pfr_deliver_rejection", w.data_ptr(), n, L.dtype_code(w), bound, r, int(MAX_REJECTION_ROUNDS),
                   c.data_ptr(), L.ptr(steps), st.data_ptr(), ws, wsb, L.stream_handle())

            def extra(bits):
                if bits & L.ST_NOPROGRESS:
                    raise RuntimeError(f"rejection resampling made no progress after {MAX_REJECTION_ROUNDS} "
                                       f"rounds; weight bound {bound} is far above every weight")
        else:
            L.call("pfr_deliver_multinomial", w.data_ptr(), n, L.dtype_code(w), L.accum_code(accum), r,
                   c.data_ptr(), L.ptr(steps), st.data_ptr(), ws, wsb, L.stream_handle())
        _raise(st, require_positive_total=True, extra=extra)  # resample_ancestors' check_weights
        c = L.to_index_dtype(c, index_dtype) if out is None else c
        return (c, int(steps.item())) if return_max_steps else c
    kw = {"rng_mode": rng_mode}
    if alg.startswith("multinomial"):
        kw["accum"] = accum
    res = resample_ancestors(w, config, rng, index_dtype=torch.int32, **kw)
    return permute_parallel(res.ancestors, return_max_steps, index_dtype=index_dtype)
