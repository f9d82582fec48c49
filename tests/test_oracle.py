"""Pin the CPU oracle against the reference: golden vectors produced by the
reference itself (tests/golden/make_golden.py) and the reference's own
known-answer tests (pkg/tests/*.py), restated.  CPU only."""

import numpy as np
import pytest

from oracle import pfr_oracle as O
from tests.golden.make_golden import ANCESTRY_CASES, WEIGHT_CASES, golden_ancestry, golden_weights


def _weights(name):
    for nm, n, seed, sigma, dtype, zeros in WEIGHT_CASES:
        if nm == name:
            return golden_weights(n, seed, sigma, dtype, zeros), seed
    raise KeyError(name)


@pytest.mark.parametrize("case", [c[0] for c in WEIGHT_CASES])
def test_weights_regenerate(golden, case):
    w, _ = _weights(case)
    assert float(w.astype(np.float64).sum()) == float(golden[f"{case}/checksum"])


@pytest.mark.parametrize("case", [c[0] for c in WEIGHT_CASES])
def test_systematic_and_permute(golden, case):
    w, seed = _weights(case)
    rs = (1000 + seed, (3, 5))
    Osys = O.systematic(w, O.systematic_offset(*rs))
    np.testing.assert_array_equal(Osys, golden[f"{case}/sys_O"])
    c, steps = O.permute(O.expand_cumulative(Osys), with_steps=True)
    np.testing.assert_array_equal(c, golden[f"{case}/sys_c"])
    assert steps == int(golden[f"{case}/sys_steps"])


@pytest.mark.parametrize("case", [c[0] for c in WEIGHT_CASES if c[1] <= 5000])
def test_resamplers_stream(golden, case):
    w, seed = _weights(case)
    seed_, ids = 1000 + seed, (3, 5)
    np.testing.assert_array_equal(np.cumsum(w), golden[f"{case}/W"])
    np.testing.assert_array_equal(O.exclusive_scan(w), golden[f"{case}/Wex"])
    np.testing.assert_array_equal(O.stratified(w, O.stratified_uniforms(seed_, ids, w.size)), golden[f"{case}/str_O"])
    np.testing.assert_array_equal(O.multinomial_stream(w, seed_, ids), golden[f"{case}/mult_a"])
    np.testing.assert_array_equal(O.multinomial_sorted(w, seed_, ids), golden[f"{case}/mser_a"])
    np.testing.assert_array_equal(O.metropolis_stream(w, 32, seed_, ids), golden[f"{case}/metro_a"])
    a, trips = O.rejection_stream(w, float(w.max()), seed_, ids)
    np.testing.assert_array_equal(a, golden[f"{case}/rej_a"])
    np.testing.assert_array_equal(trips, golden[f"{case}/rej_trips"])
    cap = float(np.median(w))
    a, trips, ow = O.rejection_stream(w, 0.0, seed_, ids, cap=cap)
    np.testing.assert_array_equal(a, golden[f"{case}/cap_a"])
    np.testing.assert_array_equal(ow, golden[f"{case}/cap_w"])
    np.testing.assert_array_equal(trips, golden[f"{case}/cap_trips"])


@pytest.mark.parametrize("case", [c[0] for c in WEIGHT_CASES if c[1] <= 5000])
@pytest.mark.parametrize("alg", ["multinomial", "multinomial-serial", "stratified", "systematic", "metropolis",
                                 "rejection", "rejection-capped"])
def test_delivery(golden, case, alg):
    w, seed = _weights(case)
    cap = float(np.median(w))
    c = O.deliver(w, alg, 2000 + seed, (7,), b=32, sup_w=float(w.max()), sup_v=cap)
    np.testing.assert_array_equal(c, golden[f"{case}/deliver/{alg}"])
    assert O.satisfies_predicate(c)


@pytest.mark.parametrize("n,seed", ANCESTRY_CASES)
@pytest.mark.parametrize("sorted_", [False, True])
def test_ancestry_golden(golden, n, seed, sorted_):
    a = golden_ancestry(n, seed, sorted_)
    tag = f"anc{n}_{'s' if sorted_ else 'u'}"
    np.testing.assert_array_equal(O.prepermute(a), golden[f"{tag}/d"])
    c, steps = O.permute(a, with_steps=True)
    np.testing.assert_array_equal(c, golden[f"{tag}/c"])
    assert steps == int(golden[f"{tag}/steps"])
    np.testing.assert_array_equal(O.permute_swaps(a), golden[f"{tag}/serial"])
    o = O.histogram(a)
    np.testing.assert_array_equal(o, golden[f"{tag}/o"])
    np.testing.assert_array_equal(np.cumsum(o), golden[f"{tag}/O"])
    np.testing.assert_array_equal(O.expand_cumulative(np.cumsum(o)), golden[f"{tag}/expand"])


def test_logweights(golden):
    lw = golden["logw/lw"]
    np.testing.assert_array_equal(O.logweights_to_weights(lw), golden["logw/w"])
    np.testing.assert_array_equal(O.logweights_to_weights(lw.astype(np.float32)), golden["logw/w32"])


def test_metropolis_steps(golden):
    for (p, e, n), b in zip(golden["msteps/args"], golden["msteps/B"]):
        assert O.metropolis_steps(float(p), None if e < 0 else float(e), int(n)) == int(b)


def test_stream_layout(golden):
    """numpy's Philox4x64-10 stream as the resamplers consume it."""
    k0, k1 = O.stream_key(4242, (1, 2, 3))
    raw = [O.philox4x64_10([blk + 1, 0, 0, 0], [k0, k1]) for blk in range(64)]
    words = [x for blk in raw for x in blk]
    u = np.array([(x >> 11) * 2.0**-53 for x in words[:64]])
    np.testing.assert_array_equal(u, golden["stream/u"])
    # integers(0, 1024): one u32 per draw, low half first; (x * 1024) >> 32
    u32 = [h for x in words[64:96] for h in (x & 0xFFFFFFFF, x >> 32)]
    np.testing.assert_array_equal([(x * 1024) >> 32 for x in u32], golden["stream/j1024"])
    derive = golden["stream/derive"]
    assert [O.derive_seed(4242, 0, 1, 2, 3), O.derive_seed(4242, 1, 1, 2, 3), O.derive_seed(0),
            O.derive_seed(2**64 - 1, 5)] == [int(x) for x in derive]


# --- the reference's known-answer tests, restated --------------------------------


def test_kat_primitives():
    np.testing.assert_array_equal(O.inclusive_scan([1.0, 2.0, 3.0]), [1, 3, 6])
    np.testing.assert_array_equal(O.exclusive_scan(np.array([1.0, 2.0, 3.0])), [0, 1, 3])
    np.testing.assert_array_equal(O.adjacent_difference([1.0, 3.0, 6.0]), [1, 2, 3])
    W = np.array([1.0, 3.0, 6.0, 10.0])
    assert O.lower_bound(W, 0.5) == 0 and O.lower_bound(W, 3.0) == 1 and O.lower_bound(W, 9.99) == 3


def test_kat_resamplers():
    np.testing.assert_array_equal(O.multinomial([1.0] * 4, [0.5, 1.5, 2.5, 3.5]), [0, 1, 2, 3])
    np.testing.assert_array_equal(O.systematic([1.0] * 4, 0.3), [1, 2, 3, 4])
    np.testing.assert_array_equal(O.systematic([1.0, 3.0], 0.9), [1, 2])
    np.testing.assert_array_equal(O.stratified([2.0, 0, 0, 0], [0.1, 0.7, 0.3, 0.9]), [4, 4, 4, 4])
    assert O.metropolis_steps(0.5, 0.005, 16) == 35
    assert O.metropolis_steps(1.0, 0.01, 4) == 17
    with pytest.raises(ValueError, match="p_star.*too small|bias bound"):
        O.metropolis_steps(0.01, 0.0001, 16)
    for s in range(5):
        np.testing.assert_array_equal(O.multinomial_stream([0.0, 0.0, 5.0, 0.0], s), [2, 2, 2, 2])
        a, _ = O.rejection_stream([0.0, 0.0, 5.0, 0.0], 5.0, s)
        np.testing.assert_array_equal(a, [2, 2, 2, 2])
    a, _ = O.rejection_stream(np.full(16, 0.7), 0.7, 0)
    np.testing.assert_array_equal(a, np.arange(16))
    np.testing.assert_array_equal(O.metropolis_stream(np.ones(64), 0, 0), np.arange(64))


def test_kat_ancestry():
    np.testing.assert_array_equal(O.expand_cumulative([2, 2, 3, 4]), [0, 0, 2, 3])
    np.testing.assert_array_equal(O.histogram([0, 0, 2, 3]), [2, 0, 1, 1])
    np.testing.assert_array_equal(O.prepermute([2, 0, 0]), [1, 3, 0])
    np.testing.assert_array_equal(O.prepermute([0, 0, 0, 0]), [0, 4, 4, 4])
    np.testing.assert_array_equal(O.permute([2, 0, 0]), [0, 0, 2])
    np.testing.assert_array_equal(O.permute_swaps([2, 0, 0]), [0, 0, 2])
    assert O.satisfies_predicate([0, 1, 2, 3]) and not O.satisfies_predicate([1, 0, 2, 1])


def test_check_weights_messages():
    with pytest.raises(ValueError, match="finite"):
        O.as_weights([1.0, np.nan])
    with pytest.raises(ValueError, match="non-negative"):
        O.as_weights([1.0, -1.0])
    with pytest.raises(ValueError, match="positive"):
        O.as_weights([0.0, 0.0])


def test_exact_metropolis_oracle_matches_matrix_power():
    rng = np.random.default_rng(3)
    for w in (rng.random(6), np.array([0.0, 1.0, 2.0, 0.0, 1.0, 3.0, 3.0])):
        n = w.size
        P = np.zeros((n, n))
        for k in range(n):
            for j in range(n):
                P[k, j] = (1.0 if w[k] == 0 else min(1.0, w[j] / w[k])) / n
            P[k, k] += 1 - P[k].sum()
        for b in (1, 3, 9):
            np.testing.assert_allclose(O.metropolis_expected_offspring(w, b),
                                       np.ones(n) @ np.linalg.matrix_power(P, b), atol=1e-13)


def test_stream_model_buffered_u32(golden):
    """The stream model the GPU rejection replay implements (pfr_rejreplay.cu):
    random() takes fresh u64s, integers() takes buffered 32-bit halves with
    Lemire redraws; an odd integer count leaves a buffered half that random()
    skips (golden: 65 draws in [0, 1000) followed by random(8))."""
    sm = O.StreamModel(4242, (1, 2, 3))
    np.testing.assert_array_equal(sm.random(64), golden["stream/u"])
    np.testing.assert_array_equal(sm.integers(1024, 64), golden["stream/j1024"])
    np.testing.assert_array_equal(sm.integers(1000, 65), golden["stream/j1000"])
    np.testing.assert_array_equal(sm.random(8), golden["stream/u2"])


def test_rejection_rounds_on_stream_model():
    """The reference's round-synchronous rejection loop consumes the stream as
    random(N), then per round integers(m) + random(m) -- restated on the
    stream model and compared with the numpy-generator oracle."""
    n = 77  # not a power of two; odd pending counts exercise the buffered half
    g = np.random.default_rng(5)
    w = np.exp(g.normal(0, 1, n))
    bound = float(w.max())
    a_ref, trips_ref = O.rejection_stream(w, bound, 9, (2,))
    sm = O.StreamModel(9, (2,))
    ratio = w / bound
    a = np.arange(n)
    trips = np.ones(n, dtype=np.int64)
    pending = np.flatnonzero(sm.random(n) > ratio)
    while pending.size:
        j = sm.integers(n, pending.size)
        beta = sm.random(pending.size)
        ok = beta <= ratio[j]
        a[pending[ok]] = j[ok]
        trips[pending] += 1
        pending = pending[~ok]
    np.testing.assert_array_equal(a, a_ref)
    np.testing.assert_array_equal(trips, trips_ref)


def test_philox4x32_vectorised_matches_scalar():
    """The vectorised Philox4x32-10 of the own-stream model equals the scalar
    restatement of csrc/pfr_rng.cuh word for word."""
    g = np.random.default_rng(5)
    c = g.integers(0, 1 << 32, (4, 64), dtype=np.uint64)
    k0, k1 = 0x9A3B1C2D, 0x01F2E3D4
    vec = O.philox4x32_10_vec(c[0], c[1], c[2], c[3], k0, k1)
    for i in range(64):
        assert [int(v[i]) for v in vec] == O.philox4x32_10([int(x) for x in c[:, i]], (k0, k1))


def test_own_rejection_model_statistics():
    """The own-stream rejection model: trip 0 proposes the slot itself, mean
    trips ~ bound / mean(v), capped weights w[a] / min(w[a], cap)."""
    g = np.random.default_rng(2)
    w = g.random(4096) + 0.5
    a, trips = O.own_rejection(w, float(w.max()), 12345)
    assert np.all(trips >= 1) and np.all(a[trips == 1] == np.flatnonzero(trips == 1))
    assert abs(trips.mean() - w.max() / w.mean()) < 0.05 * w.max() / w.mean()
    a, trips, ow = O.own_rejection(w.astype(np.float32), 1.0, 7, cap=1.0)
    np.testing.assert_array_equal(ow, np.maximum(w.astype(np.float32)[a], np.float32(1.0)) / np.float32(1.0))
