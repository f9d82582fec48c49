"""Bootstrap particle filter on the scalar linear-Gaussian model, batched over
many independent filters on the GPU (BASELINE config 5).

Mirrors pfresample.pf (pf.py:41-229): the same model, the same per-step
logic -- resample when ESS/N falls below ``ess_threshold`` through an
in-place-valid ancestry, propagate through the transition prior, weight by
the observation density, accumulate the log of the mean weighted density --
for ``filters`` independent filters at once (tile-parallel kernels over all
filters, no communication between filters; independent filters split across
GPUs by the caller).  The
propagation noise comes from the GPU's own Philox stream, so trajectories
are not the reference's draw for draw; the closed-form Kalman recursion
(pf.py:207-229, restated under ``oracle/pf_oracle.py`` -- test
infrastructure, not part of this package) is the end-to-end oracle, as in
the reference's tests.

``deliver_batched`` exposes the per-filter systematic delivery on its own.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .rng import RngStream, as_stream

__all__ = ["LinearGaussianModel", "FilterResult", "pf_run", "deliver_batched", "pf_copy_step"]


@dataclass(frozen=True)
class LinearGaussianModel:
    """x_t = coeff * x_{t-1} + trans_std * xi_t,  y_t = x_t + obs_std * eta_t,
    x_0 ~ N(initial_mean, initial_std^2) (pf.py:41-64)."""

    coeff: float = 0.0
    trans_std: float = 1.0
    obs_std: float = 1.0
    initial_mean: float = 0.0
    initial_std: float = 1.0

    def __post_init__(self):
        for name in ("trans_std", "obs_std", "initial_std"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be strictly positive")


@dataclass
class FilterResult:
    """Per-step output; arrays carry a leading filter axis for batched runs."""

    filtered_means: np.ndarray
    log_likelihood: np.ndarray | float
    ess: np.ndarray | None = field(repr=False, default=None)
    resampled: np.ndarray | None = field(repr=False, default=None)


class _PfModel(L.ctypes.Structure):
    _fields_ = [("coeff", L.ctypes.c_double), ("trans_std", L.ctypes.c_double), ("obs_std", L.ctypes.c_double),
                ("initial_mean", L.ctypes.c_double), ("initial_std", L.ctypes.c_double)]


def pf_copy_step(particles: torch.Tensor, a) -> torch.Tensor:
    """In-place gather restricted to slots with a[i] != i (pf.py:86-97).
    Requires an ancestry satisfying the in-place predicate (checked, like the
    reference's assertion)."""
    from .ancestry import copy_particles, satisfies_inplace_predicate

    if not satisfies_inplace_predicate(a):
        raise AssertionError("ancestry violates the in-place predicate")
    return copy_particles(particles, a)


_ws_pf = {}


def _workspace(key, nbytes):
    dev = L.device()
    k = (dev.index, key, L.stream_handle())  # per stream: concurrent calls on other streams
    cur = _ws_pf.get(k)
    if cur is None or cur.numel() < nbytes:
        cur = torch.empty(max(int(nbytes), 1 << 20), dtype=torch.uint8, device=dev)
        _ws_pf[k] = cur
    return cur


def pf_run(model: LinearGaussianModel, observations, n_particles: int, resampler="systematic",
           ess_threshold: float = 0.5, seed: int = 0, filters: int | None = None) -> FilterResult:
    """Run ``filters`` independent bootstrap filters (pf.py:111-204).

    ``observations``: shape (T,) (shared by every filter; ``filters``
    defaults to 1 and the result is squeezed like the reference's) or
    (filters, T).  Resampling: systematic (the batched kernels implement the
    offspring algorithm, fused into the filter's kernels; every other
    ResamplerConfig -- multinomial, stratified, Metropolis(B), rejection with
    the tracked weight bound, rejection-capped with carried importance
    weights -- runs the same filter through the library's resampling calls,
    _pf_run_general)."""
    algorithm = resampler if isinstance(resampler, str) else resampler.algorithm
    obs = np.asarray(observations, dtype=np.float64)
    squeeze = obs.ndim == 1 and filters is None
    if obs.ndim == 1:
        obs = np.broadcast_to(obs, (filters or 1, obs.size))
    if obs.ndim != 2 or obs.shape[1] == 0:
        raise ValueError("observations must be a non-empty 1-d sequence (or filters x steps)")
    if n_particles < 2:
        raise ValueError("need at least 2 particles")
    if not 0.0 <= ess_threshold <= 1.0:
        raise ValueError("ess_threshold must lie in [0, 1]")
    m_f, t_s = obs.shape
    if algorithm != "systematic":
        res = _pf_run_general(model, obs, int(n_particles), resampler, float(ess_threshold), seed)
        if squeeze:
            res = FilterResult(res.filtered_means[0], float(res.log_likelihood[0]), res.ess[0], res.resampled[0])
        return res
    dev = L.device()
    y = torch.from_numpy(np.array(obs, dtype=np.float64, order="C")).to(dev)
    means = torch.empty((m_f, t_s), dtype=torch.float64, device=dev)
    ess = torch.empty((m_f, t_s), dtype=torch.float64, device=dev)
    loglik = torch.empty(m_f, dtype=torch.float64, device=dev)
    resampled = torch.empty((m_f, t_s), dtype=torch.uint8, device=dev)
    st = L.new_status()
    nbytes = int(L.lib().pfr_pf_workspace_bytes(m_f, n_particles))
    ws = _workspace("pf", nbytes)
    k0, k1 = as_stream(RngStream(seed)).key()
    rng = L.PfrRng(k0, k1, L.RNG_PHILOX, 0)
    mdl = _PfModel(model.coeff, model.trans_std, model.obs_std, model.initial_mean, model.initial_std)
    L.call("pfr_pf_run", L.ctypes.addressof(mdl), y.data_ptr(), m_f, int(n_particles), t_s, float(ess_threshold), rng,
           means.data_ptr(), loglik.data_ptr(), ess.data_ptr(), resampled.data_ptr(), st.data_ptr(),
           ws.data_ptr(), ws.numel(), L.stream_handle())
    if L.config.check and L.read_status(st) & L.ST_NOPROGRESS:
        raise RuntimeError("weight collapse: all particle weights vanished at some step")
    res = FilterResult(means.cpu().numpy(), loglik.cpu().numpy(), ess.cpu().numpy(),
                       resampled.cpu().numpy().astype(bool))
    if squeeze:
        res = FilterResult(res.filtered_means[0], float(res.log_likelihood[0]), res.ess[0], res.resampled[0])
    return res


def _pf_run_general(model, obs, n, resampler, ess_threshold, seed) -> FilterResult:
    """pf_run (pf.py:111-204) with any ResamplerConfig, for (filters, T)
    observations.  Propagation and weighting run on the device for every
    filter at once; each filter whose ESS/N falls below the threshold
    resamples through resample_ancestors + permute_parallel and the in-place
    gather of pf_copy_step (Eq. 2).  As the reference: weights reset to 1/N
    after resampling, except rejection-capped, whose importance weights are
    carried; the rejection variants use the TRACKED weight bound (1/N after a
    reset, times sup(density) / total at each weighting), ``sup_w`` read as a
    bound on the raw observation density and ``sup_v`` as a cap on that
    scale.  Randomness: the device Philox streams (stream (seed, filter,
    purpose, step)); statistically the reference's filter."""
    from dataclasses import replace

    from .ancestry import copy_particles, permute_parallel
    from .resamplers import ResamplerConfig, resample_ancestors

    if isinstance(resampler, str):
        resampler = ResamplerConfig(algorithm=resampler)
    dev = L.device()
    m_f, t_s = obs.shape
    y = torch.from_numpy(np.ascontiguousarray(obs)).to(dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(as_stream(RngStream(seed, (1,))).key()[0] & 0x7FFFFFFFFFFFFFFF))
    density_sup = 1.0 / (model.obs_std * math.sqrt(2.0 * math.pi))
    raw_sup = resampler.sup_w if resampler.sup_w is not None else density_sup
    cap_fraction = resampler.sup_v / raw_sup if resampler.sup_v is not None else 0.5
    x = model.initial_mean + model.initial_std * torch.randn((m_f, n), generator=gen, device=dev, dtype=torch.float64)
    w = torch.full((m_f, n), 1.0 / n, dtype=torch.float64, device=dev)
    bound = np.full(m_f, 1.0 / n)
    means = torch.empty((m_f, t_s), dtype=torch.float64, device=dev)
    ess = torch.empty((m_f, t_s), dtype=torch.float64, device=dev)
    resampled = np.zeros((m_f, t_s), dtype=bool)
    loglik = torch.zeros(m_f, dtype=torch.float64, device=dev)
    for t in range(t_s):
        ess[:, t] = 1.0 / (w * w).sum(dim=1)  # compute_ess on normalised weights (diagnostics.py:54-63)
        need = torch.nonzero(ess[:, t] / n < ess_threshold).flatten().tolist()
        for m in need:
            cfg = resampler
            if resampler.algorithm == "rejection":
                cfg = replace(resampler, sup_w=float(bound[m]))
            elif resampler.algorithm == "rejection-capped":
                cfg = replace(resampler, sup_v=cap_fraction * float(bound[m]))
            out = resample_ancestors(w[m], cfg, RngStream(seed, (3, m, t)), rng_mode="philox",
                                     index_dtype=torch.int32)
            c = permute_parallel(out.ancestors, index_dtype=torch.int32)
            xm = x[m].contiguous()
            copy_particles(xm, c)
            x[m] = xm
            if out.weights is not None:
                w[m] = out.weights.to(torch.float64) / n
                bound[m] = max(1.0, 1.0 / cap_fraction) / n
            else:
                w[m] = 1.0 / n
                bound[m] = 1.0 / n
            resampled[m, t] = True
        x = model.coeff * x + model.trans_std * torch.randn((m_f, n), generator=gen, device=dev,
                                                            dtype=torch.float64)
        z = (y[:, t: t + 1] - x) / model.obs_std
        dens = torch.exp(-0.5 * z * z) * density_sup
        unnorm = w * dens
        total = unnorm.sum(dim=1)
        tot = total.cpu().numpy()
        if L.config.check and (not np.all(np.isfinite(tot)) or np.any(tot <= 0.0)):
            raise RuntimeError(f"weight collapse at step {t}: all particle weights vanished")
        loglik += torch.log(total)
        w = unnorm / total[:, None]
        bound = bound * min(raw_sup, density_sup) / tot
        means[:, t] = (w * x).sum(dim=1)
    return FilterResult(means.cpu().numpy(), loglik.cpu().numpy(), ess.cpu().numpy(), resampled)


def deliver_batched(w, rng=None, *, offsets=None, index_dtype=None, return_max_steps: bool = False):
    """Systematic delivery of each row of ``w`` (filters x N): the in-place
    ancestry c[m] of filter m with indices local to the filter, i.e. row-wise
    permute_parallel(cumulative_offspring_to_ancestors(
    systematic_cumulative_offspring(w[m]))) (resamplers.py:127-153,
    ancestry.py:69-76, 139-174).  ``offsets`` (filters,) are the filters'
    shared uniforms; otherwise each filter draws its own from ``rng``."""
    dev = L.device()
    wt = w if isinstance(w, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(w)))
    if wt.dtype not in (torch.float32, torch.float64):
        wt = wt.to(torch.float64)
    wt = wt.to(dev).contiguous()
    if wt.dim() != 2 or wt.shape[1] < 1:
        raise ValueError("w must be a (filters, N) matrix")
    m_f, n = wt.shape
    if L.config.check:
        # check_weights (diagnostics.py:38-51) for every filter's row: finite,
        # non-negative, and a positive total per row (the reference raises for
        # each filter; pfr_deliver_batched itself does not validate)
        st = L.new_status()
        L.call("pfr_check_weights", wt.data_ptr(), wt.numel(), L.dtype_code(wt), st.data_ptr(), L.stream_handle())
        L.raise_weight_errors(L.read_status(st) | L.ST_POSITIVE, "w", False)
        if not bool((wt > 0).any(dim=1).all()):
            raise ValueError("w must contain at least one strictly positive weight (in every filter's row)")
    c = torch.empty((m_f, n), dtype=torch.int32, device=dev)
    steps = torch.zeros(1, dtype=torch.int32, device=dev) if return_max_steps else None
    off = None
    if offsets is not None:
        off = torch.as_tensor(np.asarray(offsets, dtype=np.float64)).to(dev).contiguous()
        if off.numel() != m_f:
            raise ValueError("need one offset per filter")
    k0, k1 = as_stream(rng if rng is not None else RngStream(0)).key()
    r = L.PfrRng(k0, k1, L.RNG_PHILOX, 0)
    st = L.new_status()
    ws = _workspace("batched", int(L.lib().pfr_batched_workspace_bytes(m_f, n)))
    L.call("pfr_deliver_batched", wt.data_ptr(), m_f, n, L.dtype_code(wt), L.ptr(off), r, c.data_ptr(), L.ptr(steps),
           st.data_ptr(), ws.data_ptr(), ws.numel(), L.stream_handle())
    c = L.to_index_dtype(c, index_dtype)
    return (c, int(steps.item())) if return_max_steps else c
