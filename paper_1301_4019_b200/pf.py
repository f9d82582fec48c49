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
    offspring algorithm; other algorithms raise NotImplementedError)."""
    algorithm = resampler if isinstance(resampler, str) else resampler.algorithm
    if algorithm != "systematic":
        raise NotImplementedError("the batched filter resamples with the systematic algorithm")
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
