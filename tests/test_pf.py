"""Batched bootstrap particle filter (BASELINE config 5)
and the batched systematic delivery.

CPU: the closed-form Kalman oracle and the observation simulator.
GPU: the batched delivery is bit-identical per filter to the oracle's
delivery (integer weights: exact sums); the batched filter's log-likelihood
and filtered means agree with the exact Kalman filter (the reference's own
end-to-end check, test_pf.py / acceptance C10)."""

from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import pfr_oracle as orc
from oracle.pf_oracle import exact_filter, simulate_observations
from paper_1301_4019_b200.pf import LinearGaussianModel


def test_exact_filter_one_step_closed_form():
    m = LinearGaussianModel(coeff=0.5, trans_std=1.5, obs_std=0.7, initial_mean=0.3, initial_std=2.0)
    y = 1.1
    r = exact_filter(m, [y])
    p_pred = 0.25 * 4.0 + 2.25
    s = p_pred + 0.49
    gain = p_pred / s
    assert math.isclose(r.means[0], 0.15 + gain * (y - 0.15), rel_tol=1e-15)
    assert math.isclose(r.variances[0], (1 - gain) * p_pred, rel_tol=1e-15)
    assert math.isclose(r.log_likelihood, -0.5 * (math.log(2 * math.pi * s) + (y - 0.15) ** 2 / s), rel_tol=1e-15)


def test_model_validation_and_simulation():
    with pytest.raises(ValueError, match="obs_std"):
        LinearGaussianModel(obs_std=0.0)
    m = LinearGaussianModel(coeff=0.9)
    y = simulate_observations(m, 50, 3)
    assert y.shape == (50,) and np.all(np.isfinite(y))
    np.testing.assert_array_equal(y, simulate_observations(m, 50, 3))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("n", [1000, 4096, 70000])
def test_deliver_batched_matches_oracle(dtype, n):
    import paper_1301_4019_b200 as pf

    g = np.random.default_rng(n)
    filters = 6
    w = g.integers(0, 40, (filters, n)).astype(dtype)
    w[:, 0] += 1
    offsets = g.random(filters)
    c = pf.deliver_batched(w, offsets=offsets).cpu().numpy()
    for m in range(filters):
        want = orc.permute(orc.expand_cumulative(orc.systematic(w[m].astype(np.float64), float(dtype(offsets[m])))))
        np.testing.assert_array_equal(c[m], want)
        assert orc.satisfies_predicate(c[m])


@pytest.mark.gpu
def test_deliver_batched_lognormal_properties():
    import paper_1301_4019_b200 as pf

    g = np.random.default_rng(1)
    w = np.exp(g.normal(0, 1, (32, 1 << 16)))
    c, steps = pf.deliver_batched(w, pf.RngStream(5), return_max_steps=True)
    c = c.cpu().numpy()
    for m in range(0, 32, 7):
        o = np.bincount(c[m], minlength=w.shape[1])
        assert np.all(np.abs(o - w.shape[1] * w[m] / w[m].sum()) < 1.0)
        assert orc.satisfies_predicate(c[m])
    assert steps > 0


@pytest.mark.gpu
def test_batched_filter_against_kalman():
    import paper_1301_4019_b200 as pf

    model = LinearGaussianModel(coeff=0.9, trans_std=1.0, obs_std=0.8)
    y = simulate_observations(model, 60, 11)
    exact = exact_filter(model, y)
    filters, n = 128, 4096
    res = pf.pf_run(model, y, n, "systematic", 0.5, seed=3, filters=filters)
    assert res.filtered_means.shape == (filters, 60)
    assert np.all(res.ess[:, 0] == n)
    assert 0.05 < res.resampled.mean() < 0.95
    ll = res.log_likelihood
    se = ll.std(ddof=1) / math.sqrt(filters)
    # log of an unbiased likelihood estimate: bias ~ -var/2, tiny at N = 4096
    assert abs(ll.mean() - exact.log_likelihood) < 5 * se + 0.05, (ll.mean(), exact.log_likelihood, se)
    err = np.abs(res.filtered_means.mean(axis=0) - exact.means)
    assert err.max() < 0.02, err.max()
    # one filter: the reference's squeezed result
    one = pf.pf_run(model, y, 2048, seed=9)
    assert one.filtered_means.shape == (60,) and isinstance(one.log_likelihood, float)
    assert abs(one.log_likelihood - exact.log_likelihood) < 2.0


@pytest.mark.gpu
def test_batched_filter_independent_observations_and_threshold():
    import paper_1301_4019_b200 as pf

    model = LinearGaussianModel(coeff=0.5, trans_std=0.5, obs_std=0.3)
    ys = np.stack([simulate_observations(model, 20, s) for s in range(8)])
    res = pf.pf_run(model, ys, 1024, ess_threshold=0.0, seed=1)
    assert not res.resampled.any()  # threshold 0: sequential importance sampling
    res1 = pf.pf_run(model, ys, 1024, ess_threshold=1.0, seed=1)
    assert res1.resampled[:, 1:].all()
    for m in range(8):
        assert abs(res1.log_likelihood[m] - exact_filter(model, ys[m]).log_likelihood) < 3.0


@pytest.mark.gpu
@pytest.mark.parametrize("obs_std", [0.8, 0.02])
def test_batched_filter_inplace_paths_agree(monkeypatch, obs_std):
    """The global in-place pass, its unbounded fixup and the per-filter pass 3
    resolve the same ancestry, so the filters agree bit for bit (obs_std 0.02:
    degenerate weights, long chains)."""
    import paper_1301_4019_b200 as pf

    model = LinearGaussianModel(coeff=0.9, trans_std=1.0, obs_std=obs_std)
    ys = np.stack([simulate_observations(model, 12, s) for s in range(24)])
    out = []
    for path in ("0", "1", "2"):
        monkeypatch.setenv("PFR_PF_PATH", path)
        r = pf.pf_run(model, ys, 8192, ess_threshold=0.7, seed=5)
        out.append(r)
    assert out[0].resampled[:, 1:].any()
    for r in out[1:]:
        np.testing.assert_array_equal(r.filtered_means, out[0].filtered_means)
        np.testing.assert_array_equal(r.log_likelihood, out[0].log_likelihood)
        np.testing.assert_array_equal(r.ess, out[0].ess)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [4096 + 32, 3 * 4096 + 64])
def test_batched_filter_ragged_tiles_paths_agree(monkeypatch, n):
    """A ragged last tile (N % 4096 != 0, N % 32 == 0): the tile-parallel
    resample + global in-place pass equals the per-filter path bit for bit."""
    import paper_1301_4019_b200 as pf

    model = LinearGaussianModel(coeff=0.8, trans_std=0.7, obs_std=0.3)
    ys = np.stack([simulate_observations(model, 10, s) for s in range(5)])
    out = []
    for path in ("0", "1"):
        monkeypatch.setenv("PFR_PF_PATH", path)
        out.append(pf.pf_run(model, ys, n, ess_threshold=1.0, seed=2))
    assert out[0].resampled[:, 1:].all()
    np.testing.assert_array_equal(out[0].filtered_means, out[1].filtered_means)
    np.testing.assert_array_equal(out[0].log_likelihood, out[1].log_likelihood)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1000, 999])
def test_batched_filter_unaligned_sizes_track_kalman(n):
    """N % 32 != 0 (per-filter in-place pass) and odd N (scalar step path)."""
    import paper_1301_4019_b200 as pf

    model = LinearGaussianModel(coeff=0.9, trans_std=1.0, obs_std=0.8)
    y = simulate_observations(model, 30, 5)
    exact = exact_filter(model, y)
    res = pf.pf_run(model, y, n, "systematic", 0.5, seed=4, filters=64)
    assert res.resampled.any()
    ll = res.log_likelihood
    se = ll.std(ddof=1) / math.sqrt(len(ll))
    assert abs(ll.mean() - exact.log_likelihood) < 5 * se + 0.2, (ll.mean(), exact.log_likelihood, se)
    assert np.abs(res.filtered_means.mean(axis=0) - exact.means).max() < 0.1


@pytest.mark.gpu
def test_config5_full_size_against_kalman():
    """BASELINE config 5 at its full size (4096 filters x 2^16 particles,
    T = 100): the mean log-likelihood and filtered means of the batch agree
    with the exact Kalman recursion (C10, test_acceptance.py:316-347)."""
    import paper_1301_4019_b200 as pf

    model = LinearGaussianModel(coeff=0.9, trans_std=1.0, obs_std=1.0)
    y = simulate_observations(model, 100, 2024)
    exact = exact_filter(model, y)
    res = pf.pf_run(model, y, 1 << 16, "systematic", 0.5, seed=11, filters=4096)
    ll = res.log_likelihood
    se = ll.std(ddof=1) / math.sqrt(ll.size)
    assert abs(ll.mean() - exact.log_likelihood) < 5 * se + 0.01, (ll.mean(), exact.log_likelihood, se)
    assert np.abs(res.filtered_means.mean(axis=0) - exact.means).max() < 2e-3
    assert 0.2 < res.resampled.mean() < 0.8


@pytest.mark.gpu
@pytest.mark.parametrize("bad, match", [("nan", "finite"), ("neg", "non-negative"), ("zero_row", "positive")])
def test_deliver_batched_validates_every_row(bad, match):
    """a row with NaN, negative or all-zero weights raises the
    reference's ValueError instead of returning a plausible ancestry."""
    import paper_1301_4019_b200 as pf

    w = np.random.default_rng(3).random((4, 256)) + 0.1
    if bad == "nan":
        w[2, 7] = np.nan
    elif bad == "neg":
        w[1, 0] = -1.0
    else:
        w[3] = 0.0
    with pytest.raises(ValueError, match=match):
        pf.deliver_batched(w, offsets=np.full(4, 0.5))


@pytest.mark.gpu
@pytest.mark.parametrize("resampler", ["multinomial", "stratified", "metropolis", "rejection", "rejection-capped"])
def test_pf_run_every_resampler_tracks_kalman(resampler):
    """pf_run takes any ResamplerConfig (pf.py:111-204): Metropolis(B),
    rejection with the tracked weight bound, rejection-capped with carried
    importance weights, ... -- each filter's log-likelihood and filtered means
    agree with the exact Kalman recursion within Monte Carlo error."""
    import paper_1301_4019_b200 as pf
    from paper_1301_4019_b200.resamplers import ResamplerConfig

    model = LinearGaussianModel(coeff=0.9, trans_std=1.0, obs_std=0.8)
    y = simulate_observations(model, 25, 11)
    exact = exact_filter(model, y)
    # Metropolis: B from the two-state recipe (resamplers.py:350-359); a fixed
    # small B is biased on peaked weights (the paper's point)
    cfg = {"rejection-capped": ResamplerConfig("rejection-capped", sup_v=0.25)}.get(resampler,
                                                                                  ResamplerConfig(resampler))
    filters, n = 16, 2048
    res = pf.pf_run(model, y, n, cfg, 0.5, seed=5, filters=filters)
    assert res.filtered_means.shape == (filters, 25)
    assert res.resampled.any()
    ll = res.log_likelihood
    se = ll.std(ddof=1) / math.sqrt(filters)
    assert abs(ll.mean() - exact.log_likelihood) < 5 * se + 0.1, (ll.mean(), exact.log_likelihood, se)
    err = np.abs(res.filtered_means.mean(axis=0) - exact.means)
    assert err.max() < 0.08, err.max()
