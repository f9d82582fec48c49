"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle
and the reference's golden vectors.  Run on a B200 with ``-m gpu``.

Bars:
* integer functions (conversions, prepermute, permute): bit-exact, always;
* float64 systematic / stratified / multinomial / Metropolis on the reference's
  own draws (rng_mode="numpy"): bit-exact (no rounding-fragile positions at
  these sizes; checked explicitly where it matters);
* float32 scans: within a stated tolerance of an exact (float64 / fsum) scan.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import pfr_oracle as O  # noqa: E402
from tests.golden.make_golden import ANCESTRY_CASES, WEIGHT_CASES, golden_ancestry, golden_weights  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1301_4019_b200 as pf  # noqa: E402


def np_(t):
    return t.detach().cpu().numpy()


def _case(name):
    for nm, n, seed, sigma, dtype, zeros in WEIGHT_CASES:
        if nm == name:
            return golden_weights(n, seed, sigma, dtype, zeros), seed
    raise KeyError(name)


SMALL = [c[0] for c in WEIGHT_CASES if c[1] <= 5000]
ALL = [c[0] for c in WEIGHT_CASES]
F64 = [c for c in ALL if c.endswith("f64")]


# ---------------------------------------------------------------------------
# primitives


@pytest.mark.parametrize("n", [1, 2, 5, 4095, 4096, 4097, 100_000, 1 << 20])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_scan_accuracy_and_shift(n, dtype):
    g = np.random.default_rng(n)
    w = g.random(n).astype(dtype)
    W = np_(pf.inclusive_prefix_sum(w))
    Wx = np_(pf.exclusive_prefix_sum(w))
    assert W.dtype == dtype
    exact = np.cumsum(w.astype(np.float64))  # float64 fold: error << float32 ulp
    tol = (1e-12 if dtype == np.float64 else 4e-7) * np.maximum(exact, 1.0) * (1 + math.log2(n + 1))
    assert np.all(np.abs(W.astype(np.float64) - exact) <= tol)
    np.testing.assert_array_equal(Wx[1:], W[:-1])
    assert Wx[0] == 0
    assert float(pf.vector_sum(w)) == float(W[-1])
    # deterministic: bit-identical on a second run
    np.testing.assert_array_equal(np_(pf.inclusive_prefix_sum(w)), W)


def test_scan_kats():
    np.testing.assert_array_equal(np_(pf.inclusive_prefix_sum([1.0, 2.0, 3.0])), [1, 3, 6])
    np.testing.assert_array_equal(np_(pf.exclusive_prefix_sum([1.0, 2.0, 3.0])), [0, 1, 3])
    np.testing.assert_array_equal(np_(pf.adjacent_difference([1.0, 3.0, 6.0])), [1, 2, 3])
    with pytest.raises(ValueError, match="finite"):
        pf.inclusive_prefix_sum([1.0, np.nan])
    w = np.full(10, 0.1, dtype=np.float32)
    assert abs(float(pf.vector_sum(w)) - 1.0) < 1e-6
    w = np.concatenate(([2.0**24], np.ones(4096))).astype(np.float32)
    assert float(pf.vector_sum(w, accum="native")) >= 2.0**24


def test_scan_monotone_repair():
    w = np.zeros(50_000)
    w[::997] = 1e-300
    w[5] = 1.0
    W = np_(pf.inclusive_prefix_sum(w, monotone=True))
    assert np.all(np.diff(W) >= 0)


@pytest.mark.parametrize("case", SMALL)
def test_scan_matches_reference_fold(golden, case):
    w, _ = _case(case)
    W = np_(pf.inclusive_prefix_sum(w))
    ref = golden[f"{case}/W"]
    rel = 1e-13 if w.dtype == np.float64 else 2e-6
    np.testing.assert_allclose(W, ref, rtol=rel, atol=0)


def test_lower_bound_kats():
    W = np.array([1.0, 3.0, 6.0, 10.0])
    assert int(pf.lower_bound(W, 0.5)) == 0
    assert int(pf.lower_bound(W, 3.0)) == 1
    assert int(pf.lower_bound(W, 9.99)) == 3
    np.testing.assert_array_equal(np_(pf.lower_bound(np.arange(1.0, 5.0), np.array([0.5, 1.5, 2.5, 3.5]))),
                                  [0, 1, 2, 3])
    # float32 W compared in float64 (numpy promotion)
    W32 = np.array([np.float32(0.1), 1.0], dtype=np.float32)
    assert int(pf.lower_bound(W32, 0.100000002)) == int(O.lower_bound(W32, 0.100000002))


def test_lower_bound_random():
    g = np.random.default_rng(5)
    for n in (1, 7, 64, 5000):
        W = np.cumsum(g.random(n))
        q = np.concatenate([W[:-1], np.nextafter(W[:-1], 0), np.nextafter(W[:-1], np.inf), [0.0, W[-1] * 0.999]])
        np.testing.assert_array_equal(np_(pf.lower_bound(W, q)), O.lower_bound(W, q))


# ---------------------------------------------------------------------------
# weights


def test_check_weights_messages():
    with pytest.raises(ValueError, match="finite"):
        pf.check_weights([1.0, np.inf])
    with pytest.raises(ValueError, match="non-negative"):
        pf.check_weights([1.0, -2.0])
    with pytest.raises(ValueError, match="positive"):
        pf.check_weights([0.0, 0.0])
    pf.check_weights([0.0, 0.0], require_positive_total=False)
    with pytest.raises(ValueError, match="positive"):
        pf.systematic_cumulative_offspring([0.0, 0.0], pf.RngStream(0))
    with pytest.raises(ValueError, match="positive"):
        pf.multinomial_ancestors([0.0, 0.0], pf.RngStream(0))


def test_logweights(golden):
    lw = golden["logw/lw"]
    np.testing.assert_allclose(np_(pf.logweights_to_weights(lw)), golden["logw/w"], rtol=4e-16, atol=0)
    np.testing.assert_allclose(np_(pf.logweights_to_weights(lw.astype(np.float32))), golden["logw/w32"],
                               rtol=4e-7, atol=0)
    with pytest.raises(ValueError, match="NaN"):
        pf.logweights_to_weights([0.0, np.nan])
    with pytest.raises(ValueError, match="-inf"):
        pf.logweights_to_weights([-np.inf, -np.inf])


# ---------------------------------------------------------------------------
# resamplers against the reference's own draws (rng_mode="numpy")


@pytest.mark.parametrize("case", F64)
def test_systematic_bit_exact(golden, case):
    w, seed = _case(case)
    rs = pf.RngStream(1000 + seed, (3, 5))
    O_ = np_(pf.systematic_cumulative_offspring(w, rs, rng_mode="numpy"))
    np.testing.assert_array_equal(O_, golden[f"{case}/sys_O"])
    c, steps = pf.deliver(w, pf.ResamplerConfig("systematic"), rs, rng_mode="numpy", return_max_steps=True)
    np.testing.assert_array_equal(np_(c), golden[f"{case}/sys_c"])
    assert steps == int(golden[f"{case}/sys_steps"])


@pytest.mark.parametrize("case", [c for c in ALL if c.endswith("f32")])
def test_systematic_f32_within_tolerance(golden, case):
    """fp32: the reference folds in float32; we carry float64 (accum='f64').
    Stated tolerance: |O_gpu - O_ref| <= 2 slots at N <= 4096."""
    w, seed = _case(case)
    rs = pf.RngStream(1000 + seed, (3, 5))
    O_ = np_(pf.systematic_cumulative_offspring(w, rs, rng_mode="numpy")).astype(np.int64)
    ref = golden[f"{case}/sys_O"].astype(np.int64)
    assert np.abs(O_ - ref).max() <= 2
    O_n = np_(pf.systematic_cumulative_offspring(w, rs, rng_mode="numpy", accum="native")).astype(np.int64)
    assert np.abs(O_n - ref).max() <= 2


@pytest.mark.parametrize("case", [c for c in SMALL if c.endswith("f64")])
def test_stratified_multinomial_metropolis_bit_exact(golden, case):
    w, seed = _case(case)
    rs = pf.RngStream(1000 + seed, (3, 5))
    np.testing.assert_array_equal(np_(pf.stratified_cumulative_offspring(w, rs, rng_mode="numpy")),
                                  golden[f"{case}/str_O"])
    np.testing.assert_array_equal(np_(pf.multinomial_ancestors(w, rs, rng_mode="numpy")), golden[f"{case}/mult_a"])
    np.testing.assert_array_equal(np_(pf.multinomial_ancestors_serial(w, rs, rng_mode="numpy")),
                                  golden[f"{case}/mser_a"])
    if (w.size & (w.size - 1)) == 0:
        np.testing.assert_array_equal(np_(pf.metropolis_ancestors(w, 32, rs, rng_mode="numpy")),
                                      golden[f"{case}/metro_a"])
    # any N: replay the reference's draws through the ARRAYS path
    us, js = O.metropolis_draws(rs.seed, rs.ids, w.size, 32)
    np.testing.assert_array_equal(np_(pf.metropolis_ancestors(w, 32, rs, u_draws=us, j_draws=js)),
                                  golden[f"{case}/metro_a"])


@pytest.mark.parametrize("case", ["w1024_f32", "w1000_f32"])
def test_metropolis_f32_bit_exact(golden, case):
    """Metropolis has no scan: ratios rounded in float32, compared in float64,
    bit-exact in float32 too."""
    w, seed = _case(case)
    rs = pf.RngStream(1000 + seed, (3, 5))
    us, js = O.metropolis_draws(rs.seed, rs.ids, w.size, 32)
    np.testing.assert_array_equal(np_(pf.metropolis_ancestors(w, 32, rs, u_draws=us, j_draws=js)),
                                  golden[f"{case}/metro_a"])
    if (w.size & (w.size - 1)) == 0:
        np.testing.assert_array_equal(np_(pf.metropolis_ancestors(w, 32, rs, rng_mode="numpy")),
                                      golden[f"{case}/metro_a"])


def test_multinomial_injected_uniforms():
    a = pf.multinomial_ancestors([1.0, 1.0, 1.0, 1.0], pf.RngStream(0), uniforms=[0.5, 1.5, 2.5, 3.5])
    np.testing.assert_array_equal(np_(a), [0, 1, 2, 3])


@pytest.mark.parametrize("case", [c for c in SMALL if c.endswith("f64")])
@pytest.mark.parametrize("alg", ["multinomial", "multinomial-serial", "stratified", "systematic", "metropolis"])
def test_delivery_matches_reference(golden, case, alg):
    w, seed = _case(case)
    if alg == "metropolis" and (w.size & (w.size - 1)):
        pytest.skip("numpy-stream Metropolis replay needs a power-of-two N")
    cfg = pf.ResamplerConfig(alg, b=32)
    c = np_(pf.deliver(w, cfg, pf.RngStream(2000 + seed, (7,)), rng_mode="numpy"))
    np.testing.assert_array_equal(c, golden[f"{case}/deliver/{alg}"])


def test_config1_systematic_2p16_f64(golden):
    """BASELINE config 1: systematic, N=2^16 fp64, ancestors + in-place permute."""
    w, seed = _case("w65536_f64")
    rs = pf.RngStream(1000 + seed, (3, 5))
    c = np_(pf.deliver(w, pf.ResamplerConfig("systematic"), rs, rng_mode="numpy"))
    np.testing.assert_array_equal(c, golden["w65536_f64/sys_c"])


# ---------------------------------------------------------------------------
# ancestry: always bit-exact


@pytest.mark.parametrize("n,seed", ANCESTRY_CASES)
@pytest.mark.parametrize("sorted_", [False, True])
def test_ancestry_golden(golden, n, seed, sorted_):
    a = golden_ancestry(n, seed, sorted_)
    tag = f"anc{n}_{'s' if sorted_ else 'u'}"
    np.testing.assert_array_equal(np_(pf.prepermute(a)), golden[f"{tag}/d"])
    c, steps = pf.permute_parallel(a, return_max_steps=True)
    np.testing.assert_array_equal(np_(c), golden[f"{tag}/c"])
    assert steps == int(golden[f"{tag}/steps"])
    o = np_(pf.ancestors_to_offspring(a))
    np.testing.assert_array_equal(o, golden[f"{tag}/o"])
    Ocum = np_(pf.offspring_to_cumulative(o))
    np.testing.assert_array_equal(Ocum, golden[f"{tag}/O"])
    np.testing.assert_array_equal(np_(pf.cumulative_offspring_to_ancestors(Ocum)), golden[f"{tag}/expand"])
    np.testing.assert_array_equal(np_(pf.cumulative_to_offspring(Ocum)), o)
    cc, st2 = pf.permute_cumulative(Ocum, return_max_steps=True)
    c2, st3 = O.permute(O.expand_cumulative(Ocum), with_steps=True)
    np.testing.assert_array_equal(np_(cc), c2)
    assert st2 == st3


def test_ancestry_kats_and_errors():
    np.testing.assert_array_equal(np_(pf.cumulative_offspring_to_ancestors([2, 2, 3, 4])), [0, 0, 2, 3])
    np.testing.assert_array_equal(np_(pf.cumulative_offspring_to_ancestors([4, 4, 4, 4])), [0, 0, 0, 0])
    np.testing.assert_array_equal(np_(pf.prepermute([2, 0, 0])), [1, 3, 0])
    np.testing.assert_array_equal(np_(pf.permute_parallel([2, 0, 0])), [0, 0, 2])
    c, steps = pf.permute_parallel([0, 0, 0, 0], return_max_steps=True)
    assert 0 <= steps <= 4
    assert pf.satisfies_inplace_predicate([0, 1, 2, 3])
    assert not pf.satisfies_inplace_predicate([1, 0, 2, 1])
    with pytest.raises(ValueError):
        pf.cumulative_offspring_to_ancestors([2, 1, 4, 4])
    with pytest.raises(ValueError):
        pf.cumulative_offspring_to_ancestors([1, 2, 3, 5])
    with pytest.raises(ValueError):
        pf.cumulative_to_offspring([-1, 2, 3, 4])
    with pytest.raises(ValueError):
        pf.offspring_to_cumulative([2, 2, 1])
    with pytest.raises(ValueError):
        pf.offspring_to_cumulative([-1, 2, 2])
    with pytest.raises(ValueError):
        pf.permute_parallel([0, 5, 1])
    with pytest.raises(ValueError):
        pf.permute_parallel([0.5, 1.0])


def test_permute_random_many():
    g = np.random.default_rng(20240501)
    for trial in range(300):
        n = int(g.integers(1, 3000))
        a = g.integers(0, n, size=n)
        if trial % 3 == 0:
            a = np.sort(a)
        c, steps = pf.permute_parallel(a, return_max_steps=True)
        want, wsteps = O.permute(a, with_steps=True)
        np.testing.assert_array_equal(np_(c), want)
        assert steps == wsteps


@pytest.mark.parametrize("n", [300, 5000, 1 << 17])
def test_permute_long_chains_fallback(n):
    """Adversarial o = [2, 1, ..., 1, 0]: one chain of N-2 steps, far past
    the walk bound -> pointer-jumping fallback; still identical output."""
    o = np.ones(n, dtype=np.int64)
    o[0], o[-1] = 2, 0
    Ocum = np.cumsum(o)
    a = O.expand_cumulative(Ocum)
    want, wsteps = O.permute(a, with_steps=True) if n <= 5000 else (None, None)
    c1, s1 = pf.permute_parallel(a, return_max_steps=True)
    c2, s2 = pf.permute_cumulative(Ocum, return_max_steps=True)
    np.testing.assert_array_equal(np_(c1), np_(c2))
    assert s1 == s2 == n - 2
    if want is not None:
        np.testing.assert_array_equal(np_(c1), want)
        assert s1 == wsteps
    assert pf.satisfies_inplace_predicate(c1)


def test_near_uniform_weights_long_chains():
    """sigma = 0.01 weights give chains of thousands of steps."""
    g = np.random.default_rng(9)
    w = np.exp(g.normal(0, 0.01, 1 << 18))
    rs = pf.RngStream(3)
    O_ = np_(pf.systematic_cumulative_offspring(w, rs, rng_mode="numpy"))
    np.testing.assert_array_equal(O_, O.systematic(w, O.systematic_offset(3, ())))
    c, steps = pf.deliver(w, pf.ResamplerConfig("systematic"), rs, rng_mode="numpy", return_max_steps=True)
    want, wsteps = O.permute(O.expand_cumulative(O_), with_steps=True)
    np.testing.assert_array_equal(np_(c), want)
    assert steps == wsteps


def test_copy_particles():
    a = np.array([0, 0, 2, 2, 4, 1, 1, 2])
    c = O.permute(a)
    x = torch.arange(8, dtype=torch.float64, device="cuda").reshape(8, 1).repeat(1, 3).contiguous()
    pf.copy_particles(x, c)
    np.testing.assert_array_equal(np_(x)[:, 0], c.astype(np.float64))


def test_copy_particles_rejects_bad_ancestry():
    """an out-of-range c would read outside x; a length mismatch too."""
    x = torch.zeros(8, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match=r"\[0, 8\)"):
        pf.copy_particles(x, torch.tensor([0, 1, 2, 3, 4, 5, 6, 9], dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError, match="particles"):
        pf.copy_particles(torch.zeros(7, dtype=torch.float64, device="cuda"),
                          torch.arange(8, dtype=torch.int32, device="cuda"))


# ---------------------------------------------------------------------------
# large sizes: size-independent properties


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("alg", ["systematic", "stratified"])
def test_large_delivery_properties(dtype, alg):
    n = 1 << 22
    g = np.random.default_rng(11)
    w = np.exp(g.normal(0, 1, n)).astype(dtype)
    rs = pf.RngStream(77, (1,))
    wt = torch.from_numpy(w).cuda()
    cfg = pf.ResamplerConfig(alg)
    O_ = (pf.systematic_cumulative_offspring if alg == "systematic" else pf.stratified_cumulative_offspring)(
        wt, rs, index_dtype=torch.int32)
    c = pf.deliver(wt, cfg, rs, index_dtype=torch.int32)
    a_sorted = pf.cumulative_offspring_to_ancestors(O_, index_dtype=torch.int32)
    # multiset preserved, predicate holds, offspring = diff(O)
    assert torch.equal(torch.sort(c).values, a_sorted)
    assert pf.satisfies_inplace_predicate(c)
    o = pf.ancestors_to_offspring(c)
    assert torch.equal(o, pf.cumulative_to_offspring(O_))
    # stratification bound against the exact normalised weights
    m = w.astype(np.float64) * n / w.astype(np.float64).sum()
    bound = 1.0 if alg == "systematic" else 2.0
    assert np.abs(np_(o) - m).max() < bound + 1e-6


def test_large_systematic_vs_oracle_fragile_set():
    """N = 2^22 float64 against the reference formula on the reference's
    offset: mismatches may only sit at rounding-fragile positions
    (|frac(r + u) - {0,1}| within the scan's error)."""
    n = 1 << 22
    g = np.random.default_rng(12)
    w = np.exp(g.normal(0, 1, n))
    rs = pf.RngStream(5)
    O_gpu = np_(pf.systematic_cumulative_offspring(w, rs, rng_mode="numpy")).astype(np.int64)
    u = O.systematic_offset(5, ())
    O_ref = O.systematic(w, u)
    bad = np.flatnonzero(O_gpu != O_ref)
    W = np.cumsum(w)
    r = W * n / W[-1] + u
    frac = np.abs(r - np.round(r))
    assert np.all(frac[bad] < 1e-7 * n), "mismatch outside the rounding-fragile set"
    assert bad.size <= 64


# ---------------------------------------------------------------------------
# own-stream statistics (rng_mode="philox")


def _mean_offspring(fn, w, reps, seed):
    n = w.size
    counts = torch.zeros(n, dtype=torch.float64, device="cuda")
    for rep in range(reps):
        counts += fn(pf.RngStream(seed, (rep,))).double()
    return np_(counts) / reps


@pytest.mark.parametrize("alg", ["multinomial", "stratified", "systematic", "rejection", "metropolis"])
def test_unbiased_own_stream(alg):
    n, reps = 32, 4000
    g = np.random.default_rng(2024)
    w = np.exp(-0.5 * (g.normal(size=n) - 1.0) ** 2) / math.sqrt(2 * math.pi)
    wbar = w / w.sum()
    wt = torch.from_numpy(w).cuda()
    if alg in ("stratified", "systematic"):
        fn = {"stratified": pf.stratified_cumulative_offspring, "systematic": pf.systematic_cumulative_offspring}[alg]

        def draw(rs):
            return pf.cumulative_to_offspring(fn(wt, rs))
    elif alg == "multinomial":
        def draw(rs):
            return pf.ancestors_to_offspring(pf.multinomial_ancestors(wt, rs))
    elif alg == "rejection":
        def draw(rs):
            return pf.ancestors_to_offspring(pf.rejection_ancestors(wt, 1 / math.sqrt(2 * math.pi), rs))
    else:
        B = pf.metropolis_num_steps(float(wbar.max()), float(wbar.max()) * 1e-2, n)

        def draw(rs):
            return pf.ancestors_to_offspring(pf.metropolis_ancestors(wt, B, rs))
    mean = _mean_offspring(draw, w, reps, 7)
    se = np.sqrt(n * wbar * (1 - wbar) / reps)
    slack = 0.0
    if alg == "metropolis":
        exact = O.metropolis_expected_offspring(w, B)
        assert np.all(np.abs(mean - exact) < 6 * se)
        slack = float(wbar.max()) * 1e-2 * n
    assert np.all(np.abs(mean - n * wbar) < 6 * se + slack)


def test_rejection_trips_and_capped():
    n, reps = 64, 500
    g = np.random.default_rng(3)
    w = np.exp(-0.5 * (g.normal(size=n) - 1.0) ** 2) / math.sqrt(2 * math.pi)
    sup = 1 / math.sqrt(2 * math.pi)
    expected = sup * n / w.sum()
    tot = 0.0
    for rep in range(reps):
        _, trips = pf.rejection_ancestors(w, sup, pf.RngStream(43, (rep,)), return_trips=True)
        tot += float(trips.double().mean())
    assert abs(tot / reps - expected) < 0.05 * expected
    a = np_(pf.rejection_ancestors(np.full(16, 0.7), 0.7, pf.RngStream(0)))
    np.testing.assert_array_equal(a, np.arange(16))
    for s in range(5):
        np.testing.assert_array_equal(np_(pf.rejection_ancestors([0.0, 0.0, 5.0, 0.0], 5.0, pf.RngStream(s))),
                                      [2, 2, 2, 2])
    w3 = np.array([4.0, 1.0, 1.0])
    for rep in range(20):
        a, ow = pf.rejection_ancestors_capped(w3, 2.0, pf.RngStream(67, (rep,)))
        a, ow = np_(a), np_(ow)
        np.testing.assert_array_equal(ow[a == 0], 2.0)
        np.testing.assert_array_equal(ow[a != 0], 1.0)
    with pytest.raises(RuntimeError, match="no progress"):
        pf.rejection_ancestors([0.0, 0.0], 1.0, pf.RngStream(0), max_rounds=1000)


def test_metropolis_kats():
    w = np.exp(np.random.default_rng(0).normal(size=64))
    np.testing.assert_array_equal(np_(pf.metropolis_ancestors(w, 0, pf.RngStream(0))), np.arange(64))
    wz = np.array([0.0, 1.0, 2.0, 0.0, 1.0])
    for rep in range(50):
        a = np_(pf.metropolis_ancestors(wz, 20, pf.RngStream(51, (rep,))))
        assert np.all(wz[a] > 0)
    with pytest.raises(ValueError):
        pf.metropolis_ancestors(w, -1, pf.RngStream(0))


def test_zero_weights_never_ancestors():
    w = np.array([0.5, 0.0, 1.0, 0.0, 0.25, 0.0, 0.0, 2.0])
    zero = np.flatnonzero(w == 0)
    for alg in ("multinomial", "multinomial-serial", "stratified", "systematic", "rejection"):
        cfg = pf.ResamplerConfig(algorithm=alg, sup_w=2.0)
        for rep in range(30):
            out = pf.resample_ancestors(w, cfg, pf.RngStream(79, (rep,)))
            assert not np.isin(np_(out.ancestors), zero).any(), alg


def test_scale_invariance_power_of_two():
    g = np.random.default_rng(9)
    w = np.exp(g.normal(size=256)).astype(np.float32)
    s = pf.RngStream(11)
    for fn in (pf.systematic_cumulative_offspring, pf.stratified_cumulative_offspring, pf.multinomial_ancestors):
        np.testing.assert_array_equal(np_(fn(w, s)), np_(fn(w * np.float32(2.0**8), s)))
    np.testing.assert_array_equal(np_(pf.metropolis_ancestors(w, 25, s)),
                                  np_(pf.metropolis_ancestors(w * np.float32(32.0), 25, s)))
    np.testing.assert_array_equal(np_(pf.rejection_ancestors(w, 1.0 * w.max(), s)),
                                  np_(pf.rejection_ancestors(w * np.float32(4.0), 4.0 * w.max(), s)))


def test_dispatch_all_algorithms():
    g = np.random.default_rng(12)
    w = np.exp(g.normal(size=64))
    for idx, alg in enumerate(pf.ALGORITHMS):
        cfg = pf.ResamplerConfig(algorithm=alg, sup_w=float(w.max()), sup_v=float(np.median(w)))
        out = pf.resample_ancestors(w, cfg, pf.RngStream(73, (idx,)))
        a = np_(out.ancestors)
        assert a.shape == (64,) and a.min() >= 0 and a.max() < 64
        if alg == "metropolis":
            assert out.extras["B"] >= 1
        if alg.startswith("rejection"):
            assert out.extras["mean_trips"] >= 1.0
        c = pf.deliver(w, cfg, pf.RngStream(73, (idx,)))
        assert pf.satisfies_inplace_predicate(c)


def test_concurrent_streams_match_sequential():
    """Independent deliveries issued on their own streams at once (each
    (device, stream) owns its workspace and status words) give exactly the
    sequential results, for every algorithm."""
    n = 1 << 18
    g = np.random.default_rng(77)
    jobs = []
    for alg in ("multinomial", "stratified", "systematic", "metropolis", "rejection"):
        for dt in (np.float32, np.float64):
            lw = g.normal(0, 1, n)
            jobs.append((alg, torch.from_numpy(np.exp(lw - lw.max()).astype(dt)).cuda()))

    def run(alg, w, seed):
        cfg = (pf.ResamplerConfig("metropolis", b=16) if alg == "metropolis" else
               pf.ResamplerConfig("rejection", sup_w=float(w.max())) if alg == "rejection" else
               pf.ResamplerConfig(alg))
        return pf.deliver(w, cfg, pf.RngStream(seed, (3,)), index_dtype=torch.int32)

    seq = [np_(run(alg, w, k)) for k, (alg, w) in enumerate(jobs)]
    streams = [torch.cuda.Stream() for _ in jobs]
    start = torch.cuda.Event()
    start.record()
    outs = []
    for k, (alg, w) in enumerate(jobs):
        streams[k].wait_event(start)
        with torch.cuda.stream(streams[k]):
            outs.append(run(alg, w, k))
    torch.cuda.synchronize()
    for k, c in enumerate(outs):
        np.testing.assert_array_equal(np_(c), seq[k], err_msg=jobs[k][0])
    assert isinstance(pf._lib.status_all(), int)  # the rings of every stream are readable


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("alg", ["systematic", "stratified"])
@pytest.mark.parametrize("n", [1000, 1 << 16, (1 << 20) + 3])
def test_deliver_from_log_weights_is_fused_and_identical(dtype, alg, n):
    """deliver(lw, log_weights=True) equals deliver(logweights_to_weights(lw))
    element for element (the fused path computes the same exp(lw - max))."""
    g = np.random.default_rng(n)
    lw = (g.normal(0, 2.0, n) - 30.0).astype(dtype)
    lw[::53] = -np.inf
    lwt = torch.from_numpy(lw).cuda()
    cfg = pf.ResamplerConfig(alg)
    fused = pf.deliver(lwt, cfg, pf.RngStream(4, (n,)), log_weights=True, index_dtype=torch.int32)
    two = pf.deliver(pf.logweights_to_weights(lwt), cfg, pf.RngStream(4, (n,)), index_dtype=torch.int32)
    np.testing.assert_array_equal(np_(fused), np_(two))
    assert O.satisfies_predicate(np_(fused))


def test_deliver_from_log_weights_errors_and_other_algorithms():
    cfg = pf.ResamplerConfig("systematic")
    with pytest.raises(ValueError, match=r"NaN or \+inf"):
        pf.deliver(torch.tensor([0.0, float("nan"), 1.0], device="cuda"), cfg, pf.RngStream(0), log_weights=True)
    with pytest.raises(ValueError, match="all log-weights are -inf"):
        pf.deliver(torch.full((5,), float("-inf"), device="cuda", dtype=torch.float64), cfg, pf.RngStream(0),
                   log_weights=True)
    lw = torch.from_numpy(np.random.default_rng(1).normal(0, 1, 4096)).cuda()
    mh = pf.ResamplerConfig("metropolis", b=8)
    a = pf.deliver(lw, mh, pf.RngStream(2), log_weights=True)
    b = pf.deliver(pf.logweights_to_weights(lw), mh, pf.RngStream(2))
    np.testing.assert_array_equal(np_(a), np_(b))


def test_multinomial_validates_inside_its_scan():
    """multinomial_ancestors has no separate check pass: the weight scan
    reports check_weights' flags with the reference's messages."""
    with pytest.raises(ValueError, match="non-negative"):
        pf.multinomial_ancestors(np.array([1.0, -1.0, 2.0]), pf.RngStream(0))
    with pytest.raises(ValueError, match="finite"):
        pf.multinomial_ancestors(np.array([1.0, np.inf, 2.0]), pf.RngStream(0))
    with pytest.raises(ValueError, match="positive"):
        pf.multinomial_ancestors(np.zeros(5), pf.RngStream(0))
    a = np_(pf.multinomial_ancestors(np.array([0.0, 0.0, 5.0, 0.0]), pf.RngStream(1)))
    np.testing.assert_array_equal(a, [2, 2, 2, 2])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_metropolis_own_stream_validates_in_kernel(dtype):
    """Own-stream Metropolis has no separate check pass: the chains' first
    reads report check_weights' flags (all-zero weights are allowed, as in
    the reference)."""
    with pytest.raises(ValueError, match="non-negative"):
        pf.metropolis_ancestors(np.array([1.0, -1.0, 2.0, 3.0], dtype=dtype), 4, pf.RngStream(0))
    with pytest.raises(ValueError, match="finite"):
        pf.metropolis_ancestors(np.array([1.0, np.nan, 2.0, 3.0], dtype=dtype), 4, pf.RngStream(0))
    a = np_(pf.metropolis_ancestors(np.zeros(8, dtype=dtype), 4, pf.RngStream(0)))
    assert a.min() >= 0 and a.max() < 8
    big = np.exp(np.random.default_rng(3).normal(0, 1, 100003)).astype(dtype)
    big[77777] = -0.5
    with pytest.raises(ValueError, match="non-negative"):
        pf.metropolis_ancestors(big, 2, pf.RngStream(1))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_rejection_validates_in_kernel(dtype):
    """Rejection has no separate check pass: each slot's first trip (which
    proposes the slot itself) reports check_weights' flags."""
    with pytest.raises(ValueError, match="non-negative"):
        pf.rejection_ancestors(np.array([1.0, -1.0, 2.0, 3.0], dtype=dtype), 3.0, pf.RngStream(0))
    w = np.exp(np.random.default_rng(4).normal(0, 1, 50001)).astype(dtype)
    a, trips = pf.rejection_ancestors(w, float(w.max()), pf.RngStream(2), return_trips=True)
    assert np_(trips).min() >= 1 and O.satisfies_predicate(O.permute(np_(a)))
    w[31337] = -1.0
    with pytest.raises(ValueError, match="non-negative"):
        pf.rejection_ancestors(w, float(w.max()), pf.RngStream(2))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [1000, 1 << 16, (1 << 20) + 5])
def test_fused_metropolis_delivery_equals_two_calls(dtype, n):
    """deliver(metropolis) in the own stream (claims made by the chains)
    equals permute_parallel(metropolis_ancestors(...)) element for element,
    max steps included."""
    g = np.random.default_rng(n)
    w = torch.from_numpy(np.exp(g.normal(0, 1.5, n)).astype(dtype)).cuda()
    cfg = pf.ResamplerConfig("metropolis", b=12)
    c, s = pf.deliver(w, cfg, pf.RngStream(8, (n,)), return_max_steps=True, index_dtype=torch.int32)
    a = pf.metropolis_ancestors(w, 12, pf.RngStream(8, (n,)), index_dtype=torch.int32)
    c2, s2 = pf.permute_parallel(a, return_max_steps=True, index_dtype=torch.int32)
    np.testing.assert_array_equal(np_(c), np_(c2))
    assert s == s2


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n, sigma, b, zeros", [(1 << 22, 1.0, 32, 0.0), (70001, 1.0, 7, 0.3), (1 << 20, 0.3, 5, 0.0),
                                                (4096, 2.0, 32, 0.5)])
def test_fused_metropolis_delivery_more_cases(dtype, n, sigma, b, zeros):
    """The fused Metropolis delivery (claims made by the chains) against the
    plain chains + permute at more shapes: 2^22, odd N and odd B, zero
    weights, flat and peaked weights."""
    g = np.random.default_rng(n + b)
    wn = np.exp(g.normal(0, sigma, n))
    wn[g.random(n) < zeros] = 0.0
    w = torch.from_numpy(wn.astype(dtype)).cuda()
    cfg = pf.ResamplerConfig("metropolis", b=b)
    c, s = pf.deliver(w, cfg, pf.RngStream(21, (n,)), return_max_steps=True, index_dtype=torch.int32)
    a = pf.metropolis_ancestors(w, b, pf.RngStream(21, (n,)), index_dtype=torch.int32)
    c2, s2 = pf.permute_parallel(a, return_max_steps=True, index_dtype=torch.int32)
    np.testing.assert_array_equal(np_(c), np_(c2))
    assert s == s2


@pytest.mark.parametrize("alg", ["systematic", "metropolis"])
def test_config4_full_size_properties(alg):
    """BASELINE config 4 at its full size, N = 2^28 float32 on one GPU:
    size-independent properties of the delivered ancestry (in-place
    predicate, multiset = the resampler's ancestry; systematic: offspring
    within 1 of N w/W)."""
    n = 1 << 28
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    lw = torch.randn(n, device="cuda", generator=g)
    w = torch.exp(lw - lw.max())
    del lw
    if alg == "systematic":
        rs = pf.RngStream(9)
        O_ = pf.systematic_cumulative_offspring(w, rs, index_dtype=torch.int32)
        c = pf.deliver(w, pf.ResamplerConfig("systematic"), rs, index_dtype=torch.int32)
        o = pf.ancestors_to_offspring(c)
        assert torch.equal(o, pf.cumulative_to_offspring(O_, index_dtype=torch.int32))
        m = w.double() * (n / w.double().sum())
        assert float((o.double() - m).abs().max()) < 1.0 + 1e-6
        del O_, m
    else:
        rs = pf.RngStream(10)
        a = pf.metropolis_ancestors(w, 4, rs, index_dtype=torch.int32)
        c = pf.deliver(w, pf.ResamplerConfig("metropolis", b=4), rs, index_dtype=torch.int32)
        assert torch.equal(pf.ancestors_to_offspring(c), pf.ancestors_to_offspring(a))
        del a
    assert pf.satisfies_inplace_predicate(c)
    del c, w
    torch.cuda.empty_cache()


def _rej_weights(kind, n, dtype, seed):
    g = np.random.default_rng(seed)
    if kind == "lognormal1":
        w = np.exp(g.normal(0, 1, n))
    elif kind == "lognormal2":
        w = np.exp(g.normal(0, 2, n))
    elif kind == "uniform":
        w = g.random(n)
    elif kind == "spikes":  # a few large weights, the rest tiny or zero
        w = g.random(n) * 1e-3
        w[g.integers(0, n, 5)] = 1.0
        w[g.random(n) < 0.3] = 0.0
    else:
        raise KeyError(kind)
    return w.astype(dtype)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [4096, 1 << 16])
@pytest.mark.parametrize("kind", ["lognormal1", "lognormal2", "uniform", "spikes"])
@pytest.mark.parametrize("capped", [False, True])
def test_rejection_own_stream_matches_model(dtype, n, kind, capped):
    """Own-stream rejection, bit for bit against the oracle's model of the
    stream (ancestors, trip counts, capped importance weights)."""
    w = _rej_weights(kind, n, dtype, n + len(kind))
    rs = pf.RngStream(31, (n, int(capped)))
    key0 = rs.key()[0]
    if capped:
        cap = float(np.quantile(w, 0.9))
        a, ow, trips = pf.rejection_ancestors_capped(w, cap, rs, return_trips=True)
        wa, wt, wo = O.own_rejection(w, cap, key0, cap=cap)
        np.testing.assert_array_equal(np_(ow), wo)
    else:
        bound = float(w.max()) * (1.5 if kind == "lognormal2" else 1.0)
        a, trips = pf.rejection_ancestors(w, bound, rs, return_trips=True)
        wa, wt = O.own_rejection(w, bound, key0)
    np.testing.assert_array_equal(np_(a), wa)
    np.testing.assert_array_equal(np_(trips), wt)


_TABLE_AB = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1301_4019_b200 as pf
out = {}
# g = 1, 2, 4 weights per table bit; non-power-of-two N (Lemire redraws)
for n in (1 << 20, 1000003, 1 << 21, 3 << 20):
    for dt in (np.float32, np.float64):
        g = np.random.default_rng(n)
        w = np.exp(g.normal(0, 0.8, n)).astype(dt)
        w[g.random(n) < 0.2] = 0
        a, t = pf.rejection_ancestors(w, float(w.max()), pf.RngStream(9, (n,)), return_trips=True)
        a2, ow, t2 = pf.rejection_ancestors_capped(w, float(np.quantile(w, 0.95)), pf.RngStream(10, (n,)),
                                                   return_trips=True)
        k = f"{n}_{np.dtype(dt).name}"
        out[k + "_a"], out[k + "_t"] = a.cpu().numpy(), t.cpu().numpy()
        out[k + "_ca"], out[k + "_cw"], out[k + "_ct"] = a2.cpu().numpy(), ow.cpu().numpy(), t2.cpu().numpy()
np.savez(sys.argv[1], **out)
"""


def test_rejection_table_on_off_identical(tmp_path):
    """The certain-reject table (DESIGN 3.4) only skips gathers whose outcome
    is decided: ancestors, trips and capped weights equal the plain kernel's
    (PFR_REJ_TABLE=0) for g = 1, 2, 4 weights per bit, power-of-two and odd N,
    zero weights -- two processes, the switch is read once per process."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for flag in ("1", "0"):
        f = tmp_path / f"t{flag}.npz"
        env = dict(os.environ, PFR_REJ_TABLE=flag)
        subprocess.run([sys.executable, "-c", _TABLE_AB, str(f)], cwd=root, env=env, check=True, timeout=600)
        res.append(np.load(f))
    assert set(res[0].files) == set(res[1].files) and len(res[0].files) == 40
    for k in res[0].files:
        np.testing.assert_array_equal(res[0][k], res[1][k], err_msg=k)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("alg", ["rejection", "multinomial"])
@pytest.mark.parametrize("n", [1, 1000, 4097, (1 << 20) + 5])
def test_fused_rejection_multinomial_delivery_equals_two_calls(dtype, alg, n):
    """deliver(rejection / multinomial) in the own stream makes the permute's
    claims inside the resampler: element for element (and max steps) the
    same as permute_parallel(resample_ancestors(...))."""
    g = np.random.default_rng(n + 3)
    wn = np.exp(g.normal(0, 1.0, n))
    wn[g.random(n) < 0.1] = 0.0
    wn[0] = 1.0
    w = torch.from_numpy(wn.astype(dtype)).cuda()
    cfg = pf.ResamplerConfig(alg, sup_w=float(w.max()) if alg == "rejection" else None)
    c, s = pf.deliver(w, cfg, pf.RngStream(4, (n,)), return_max_steps=True, index_dtype=torch.int32)
    a = pf.resample_ancestors(w, cfg, pf.RngStream(4, (n,)), index_dtype=torch.int32).ancestors
    c2, s2 = pf.permute_parallel(a, return_max_steps=True, index_dtype=torch.int32)
    np.testing.assert_array_equal(np_(c), np_(c2))
    assert s == s2
    assert O.satisfies_predicate(np_(c))


@pytest.mark.parametrize("alg", ["rejection", "multinomial"])
def test_fused_delivery_validates(alg):
    with pytest.raises(ValueError, match="non-negative"):
        pf.deliver(np.array([1.0, -1.0, 2.0, 3.0]), pf.ResamplerConfig(alg, sup_w=3.0 if alg == "rejection" else None),
                   pf.RngStream(0))
    with pytest.raises(ValueError, match="positive"):
        pf.deliver(np.zeros(8), pf.ResamplerConfig(alg, sup_w=1.0 if alg == "rejection" else None), pf.RngStream(0))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("kind", ["two_spikes", "mostly_zero", "ramp"])
def test_own_stream_multinomial_long_weight_runs(dtype, kind):
    """The own-stream multinomial merge when a uniform tile's W run does not
    fit shared memory (flat stretches of zero weights: the global-memory
    path): the ancestry is sorted, selects only positive weights, and its
    counts follow N w / W."""
    n = (1 << 18) + 77
    g = np.random.default_rng(len(kind))
    if kind == "two_spikes":
        w = np.zeros(n)
        w[0], w[-1] = 1.0, 1.0
    elif kind == "mostly_zero":
        w = np.zeros(n)
        idx = g.choice(n, 300, replace=False)
        w[idx] = g.random(300) + 0.5
    else:
        w = np.linspace(0.0, 1.0, n) ** 8
    w = w.astype(dtype)
    for fused in (False, True):
        if fused:
            c = np_(pf.deliver(w, pf.ResamplerConfig("multinomial"), pf.RngStream(6), index_dtype=torch.int64))
            assert O.satisfies_predicate(c)
            a = np.sort(c)
        else:
            a = np_(pf.multinomial_ancestors(w, pf.RngStream(6), index_dtype=torch.int64))
            assert np.all(np.diff(a) >= 0)
        assert np.all(w[a] > 0)
        cnt = np.bincount(a, minlength=n).astype(np.float64)
        expect = n * w.astype(np.float64) / w.astype(np.float64).sum()
        sd = np.sqrt(np.maximum(expect, 1.0))
        assert np.all(np.abs(cnt - expect) < 7 * sd + 1)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [4096, 70000])
def test_delivery_long_chain_goes_to_the_rare_path(dtype, n):
    """w = (2, 1, ..., 1, 0): O = (2, 3, ..., N, N), one loser chain of
    length N-2 -- past the resolve kernel's bounds (per-chain steps when
    max_steps is requested, the drain's pass count otherwise), so the rare
    path resolves it: both calls equal the oracle's delivery."""
    w = np.ones(n)
    w[0], w[-1] = 2.0, 0.0
    w = w.astype(dtype)
    # O does not depend on the offset here: floor(j + 2 + u) = j + 2 for any u
    want = O.permute(O.expand_cumulative(O.systematic(w.astype(np.float64), 0.5)))
    cfg = pf.ResamplerConfig("systematic")
    c_track, steps = pf.deliver(w, cfg, pf.RngStream(0), return_max_steps=True, index_dtype=torch.int64)
    c_plain = pf.deliver(w, cfg, pf.RngStream(0), index_dtype=torch.int64)
    np.testing.assert_array_equal(np_(c_track), want)
    np.testing.assert_array_equal(np_(c_plain), want)
    assert steps >= n - 2
