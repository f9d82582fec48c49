"""Config 3 (BASELINE.json): weight-variance sweep, statistics of the GPU's own
Philox stream at scale.

* Metropolis(B) bias against the EXACT expected offspring 1^T P^B of the
  independence sampler (oracle
  metropolis_expected_offspring) -- every chain is independent, so the
  offspring count of particle i is a sum of N independent Bernoullis whose
  variance is bounded by the binomial one (conservative z-scores).
* Rejection: mean trips per slot equal N * sup_w / sum(w) in expectation
  (trip 0 proposes the slot itself, resamplers.py:291-294), and offspring are
  unbiased (E[o_i] = N w_i / sum(w)).
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import pfr_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

import paper_1301_4019_b200 as pf  # noqa: E402


def lognormal(n, sigma, seed):
    g = np.random.default_rng(seed)
    lw = g.normal(0.0, sigma, n)
    return np.exp(lw - lw.max())


def mean_offspring(draw, n, reps, seed):
    acc = torch.zeros(n, dtype=torch.float64, device="cuda")
    for r in range(reps):
        acc += pf.ancestors_to_offspring(draw(pf.RngStream(seed, (r,)))).to(torch.float64)
    return (acc / reps).cpu().numpy()


@pytest.mark.parametrize("sigma", [0.5, 1.0, 2.0])
@pytest.mark.parametrize("steps", [1, 4, 16])
def test_metropolis_bias_matches_exact_curve(sigma, steps):
    n, reps = 4096, 300
    w = lognormal(n, sigma, 11)
    wt = torch.from_numpy(w).cuda()
    exact = O.metropolis_expected_offspring(w, steps)
    assert abs(exact.sum() - n) < 1e-6 * n
    mean = mean_offspring(lambda rs: pf.metropolis_ancestors(wt, steps, rs), n, reps, 100 + steps)
    # o_i is a sum of N independent Bernoullis (chains start at different
    # indices, so not identically distributed): its variance is at most the
    # binomial N p (1 - p) -- the z-scores below are conservative
    p = np.clip(exact / n, 1e-300, 1.0)
    se = np.sqrt(n * p * (1 - p) / reps)
    z = (mean - exact) / se
    assert np.max(np.abs(z)) < 5.5, float(np.max(np.abs(z)))
    assert np.mean(z ** 2) < 1.15, float(np.mean(z ** 2))
    # the bias the paper discusses: E[o_max] / (N p_max) < 1 for small B
    i = int(np.argmax(w))
    ratio = exact[i] / (n * w[i] / w.sum())
    assert 0.0 < ratio <= 1.0 + 1e-9


@pytest.mark.parametrize("sigma", [0.5, 1.0, 1.5])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_rejection_acceptance_and_unbiasedness(sigma, dtype):
    n, reps = 4096, 200
    w = lognormal(n, sigma, 5).astype(dtype)
    wt = torch.from_numpy(w).cuda()
    sup = float(w.max())
    expected_trips = n * sup / float(w.astype(np.float64).sum())
    trips_mean = []
    acc = torch.zeros(n, dtype=torch.float64, device="cuda")
    for r in range(reps):
        a, trips = pf.rejection_ancestors(wt, sup, pf.RngStream(77, (r,)), return_trips=True)
        trips_mean.append(float(trips.double().mean()))
        acc += pf.ancestors_to_offspring(a).to(torch.float64)
    tm = np.mean(trips_mean)
    # per-slot trips: 1 + Geometric(acc) after a rejected self-proposal; the mean over
    # N * reps slots has a relative standard error well below 1% here
    assert abs(tm / expected_trips - 1.0) < 0.02, (tm, expected_trips)
    mean = (acc / reps).cpu().numpy()
    wbar = w.astype(np.float64) / w.astype(np.float64).sum()
    se = np.sqrt(n * wbar * (1 - wbar) / reps)
    z = (mean - n * wbar) / se
    assert np.max(np.abs(z)) < 5.5


@pytest.mark.parametrize("alg", ["systematic", "stratified"])
def test_offspring_stratification_bounds(alg):
    """|o_i - N w_i / W| < 1 (systematic) and < 2 (stratified) on every draw
    (test_acceptance.py C4 analogue, SPEC criterion 4)."""
    n = 1 << 16
    w = lognormal(n, 1.0, 9)
    fn = pf.systematic_cumulative_offspring if alg == "systematic" else pf.stratified_cumulative_offspring
    target = n * w / w.sum()
    worst = 0.0
    for r in range(20):
        o = pf.cumulative_to_offspring(fn(w, pf.RngStream(3, (r,)))).cpu().numpy()
        worst = max(worst, float(np.max(np.abs(o - target))))
    assert worst < (1.0 if alg == "systematic" else 2.0), worst
