"""Property-based and chi-square tests on the GPU path (the
reference's Hypothesis properties, test_ancestry.py:29-32,143-148 and
test_primitives.py:147-158, re-targeted at the CUDA functions; its
statistical tests restated as chi-square goodness of fit).

Properties are checked against the oracle (tests/ only) on random small
inputs; the chi-square tests use the GPU's own Philox stream."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
hypothesis = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, assume, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402
from scipy import stats  # noqa: E402

from oracle import pfr_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1301_4019_b200 as pf  # noqa: E402

_settings = settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])


@st.composite
def ancestries(draw, max_n=256):
    """Random ancestry vectors, half of them sorted (test_ancestry.py:29-32)."""
    n = draw(st.integers(1, max_n))
    a = draw(st.lists(st.integers(0, n - 1), min_size=n, max_size=n))
    if draw(st.booleans()):
        a = sorted(a)
    return np.array(a, dtype=np.int64)


def np_(t):
    return t.detach().cpu().numpy()


@_settings
@given(ancestries())
def test_permute_properties(a):
    """Predicate, multiset, termination and the reference's exact vector
    (ancestry.py:97-101, 139-174)."""
    c, steps = pf.permute_parallel(a, return_max_steps=True)
    c = np_(c)
    want, wsteps = O.permute(a, with_steps=True)
    np.testing.assert_array_equal(c, want)
    assert steps == wsteps
    assert O.satisfies_predicate(c)
    np.testing.assert_array_equal(np.sort(c), np.sort(a))
    assert pf.satisfies_inplace_predicate(c)


@_settings
@given(ancestries())
def test_conversion_round_trips(a):
    """ancestors -> offspring -> cumulative -> sorted ancestors, and back."""
    o = np_(pf.ancestors_to_offspring(a))
    np.testing.assert_array_equal(o, O.histogram(a))
    Ocum = np_(pf.offspring_to_cumulative(o))
    np.testing.assert_array_equal(Ocum, np.cumsum(o))
    np.testing.assert_array_equal(np_(pf.cumulative_offspring_to_ancestors(Ocum)), np.sort(a))
    np.testing.assert_array_equal(np_(pf.cumulative_to_offspring(Ocum)), o)
    np.testing.assert_array_equal(np_(pf.permute_cumulative(Ocum)), O.permute(np.sort(a)))


@_settings
@given(st.lists(st.floats(0.0, 10.0, allow_nan=False), min_size=1, max_size=300),
       st.lists(st.floats(0.0, 1.0, allow_nan=False, exclude_max=True), min_size=1, max_size=64))
def test_lower_bound_matches_linear_scan(w, fr):
    """smallest j with W[j] >= u, clamped to N-1 (primitives.py:91-106)
    against a linear scan (test_primitives.py:147-158)."""
    W = np.cumsum(np.asarray(w, dtype=np.float64))
    u = np.asarray(fr) * W[-1]
    got = np_(pf.lower_bound(W, u))
    lin = np.array([min(next((j for j in range(W.size) if W[j] >= x), W.size - 1), W.size - 1) for x in u])
    np.testing.assert_array_equal(got, lin)


@_settings
@given(st.lists(st.floats(0.0, 1e6, allow_nan=False), min_size=1, max_size=2000).filter(lambda v: sum(v) > 0),
       st.sampled_from(["float32", "float64"]))
def test_systematic_offspring_properties(w, dtype):
    """O non-decreasing, ends at N, per-parent counts within 1 of N w/W
    (systematic_cumulative_offspring, resamplers.py:127-153)."""
    w = np.asarray(w, dtype=dtype)
    assume(w.max() > 0)  # float32 flushes the tiniest draws to zero
    n = w.size
    O_ = np_(pf.systematic_cumulative_offspring(w, pf.RngStream(len(w))))
    assert O_[-1] == n and np.all(np.diff(O_) >= 0)
    o = np.diff(np.concatenate(([0], O_)))
    exp = n * w.astype(np.float64) / w.astype(np.float64).sum()
    assert np.all(np.abs(o - exp) < 1.0 + 1e-6 * n)


# ---------------------------------------------------------------------------
# chi-square goodness of fit of the aggregated offspring counts, own stream

_N, _R = 64, 4000


def _weights(seed):
    g = np.random.default_rng(seed)
    w = np.exp(g.normal(0, 1.0, _N))
    w[::9] = 0.0  # zero weights: never chosen
    return w


def _counts(fn, w):
    total = np.zeros(_N)
    for r in range(_R):
        total += O.histogram(np_(fn(r)))
    return total


@pytest.mark.parametrize("alg", ["multinomial", "stratified", "systematic", "rejection"])
def test_offspring_chi_square(alg):
    """Summed offspring over R replicates against R N w/W: chi-square p >= 1e-3
    (the reference's unbiasedness, test_resamplers.py:62-72,104-117; the
    variance-reducing resamplers only make the statistic smaller)."""
    w = _weights(11)
    wt = torch.from_numpy(w).cuda()
    cfg = pf.ResamplerConfig(alg, sup_w=float(w.max()) if alg == "rejection" else None)
    counts = _counts(lambda r: pf.resample_ancestors(wt, cfg, pf.RngStream(r, (7,))).ancestors, w)
    exp = _R * _N * w / w.sum()
    assert np.all(counts[exp == 0] == 0)
    m = exp > 0
    chi2 = float(((counts[m] - exp[m]) ** 2 / exp[m]).sum())
    p = stats.chi2.sf(chi2, int(m.sum()) - 1)
    assert p >= 1e-3, (alg, chi2, p)


@pytest.mark.parametrize("b", [2, 8, 64])
def test_metropolis_chi_square_against_exact(b):
    """Metropolis offspring against its exact expectation 1^T P^B (SURVEY
    A.9), not N w/W: chi-square p >= 1e-3 at every B."""
    w = _weights(12)
    wt = torch.from_numpy(w).cuda()
    counts = _counts(lambda r: pf.metropolis_ancestors(wt, b, pf.RngStream(r, (b,))), w)
    exp = _R * O.metropolis_expected_offspring(w, b)
    m = exp > 1e-9
    assert np.all(counts[~m] == 0)
    chi2 = float(((counts[m] - exp[m]) ** 2 / exp[m]).sum())
    p = stats.chi2.sf(chi2, int(m.sum()) - 1)
    assert p >= 1e-3, (b, chi2, p)
