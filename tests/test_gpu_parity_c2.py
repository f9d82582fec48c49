"""Parity at the headline configuration (BASELINE configs[1]: all five
resamplers, N = 2^20, float32 and float64) and at the north-star size
(N = 2^24 float32), element by element against the oracle.

The oracle (oracle/pfr_oracle.py) reproduces the reference bit for bit
(pinned by tests/golden).  All GPU calls go through the C ABI
with the reference's own draws (rng_mode="numpy").

Bars:
* accum="serial" (the reference's np.cumsum fold performed on the GPU):
  systematic / stratified / multinomial ancestries, offspring and deliveries
  are BIT-EXACT in float32 and float64 at any N;
* Metropolis(B=32) and rejection (round-synchronous replay): bit-exact in
  float32 and float64 (no scan involved);
* the default accum="f64" (deterministic parallel scan carried in float64):
  float64 bit-exact at 2^20 (no rounding-fragile position); float32 within
  the stated tolerance -- positions within 1 of a float64 fold of the same
  float32 weights, so the distance to the reference's float32 output is the
  reference's own float32 drift plus at most 1.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import pfr_oracle as O  # noqa: E402
from tests.golden.make_golden import WEIGHT_CASES, golden_weights  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1301_4019_b200 as pf  # noqa: E402

N20 = 1 << 20
DT = {"f32": np.float32, "f64": np.float64}


def np_(t):
    return t.detach().cpu().numpy()


def _w(n, dt, seed=20):
    return golden_weights(n, seed, 1.0, DT[dt])


@pytest.fixture(scope="module")
def c2():
    return {dt: _w(N20, dt, 20 + i) for i, dt in enumerate(DT)}


# ---------------------------------------------------------------------------
# serial fold: np.cumsum bit for bit


@pytest.mark.parametrize("dt", list(DT))
@pytest.mark.parametrize("n", [1, 5, 4095, 4097, N20])
def test_serial_scan_is_cumsum(dt, n):
    w = _w(n, dt, 3)
    got = np_(pf.inclusive_prefix_sum(w, accum="serial"))
    np.testing.assert_array_equal(got, np.cumsum(w))
    ex = np_(pf.exclusive_prefix_sum(w, accum="serial"))
    np.testing.assert_array_equal(ex[1:], np.cumsum(w[:-1]))
    assert ex[0] == 0
    assert float(pf.vector_sum(w, accum="serial")) == float(np.cumsum(w)[-1])


@pytest.mark.parametrize("dt", list(DT))
def test_c2_systematic_stratified_serial_bit_exact(c2, dt):
    w = c2[dt]
    rs = pf.RngStream(1001, (3, 5))
    O_sys = np_(pf.systematic_cumulative_offspring(w, rs, rng_mode="numpy", accum="serial"))
    np.testing.assert_array_equal(O_sys, O.systematic(w, O.systematic_offset(1001, (3, 5))))
    O_str = np_(pf.stratified_cumulative_offspring(w, rs, rng_mode="numpy", accum="serial"))
    np.testing.assert_array_equal(O_str, O.stratified(w, O.stratified_uniforms(1001, (3, 5), w.size)))


@pytest.mark.parametrize("dt", list(DT))
def test_c2_multinomial_serial_bit_exact(c2, dt):
    w = c2[dt]
    rs = pf.RngStream(1002, (1,))
    a = np_(pf.multinomial_ancestors(w, rs, rng_mode="numpy", accum="serial"))
    np.testing.assert_array_equal(a, O.multinomial_stream(w, 1002, (1,)))


@pytest.mark.parametrize("dt", list(DT))
def test_c2_metropolis_bit_exact(c2, dt):
    w = c2[dt]
    a = np_(pf.metropolis_ancestors(w, 32, pf.RngStream(1003, (2,)), rng_mode="numpy"))
    np.testing.assert_array_equal(a, O.metropolis_stream(w, 32, 1003, (2,)))


@pytest.mark.parametrize("dt", list(DT))
def test_c2_rejection_bit_exact(c2, dt):
    """Round-synchronous replay of resamplers.py:282-310 on the reference's
    stream: ancestry AND trip counts equal, sup_w = max w (~106 trips/slot,
    ~1,900 rounds)."""
    w = c2[dt]
    a, trips = pf.rejection_ancestors(w, float(w.max()), pf.RngStream(1004, (4,)), return_trips=True,
                                      rng_mode="numpy")
    a_ref, trips_ref = O.rejection_stream(w, float(w.max()), 1004, (4,))
    np.testing.assert_array_equal(np_(a), a_ref)
    np.testing.assert_array_equal(np_(trips), trips_ref)


@pytest.mark.parametrize("dt", list(DT))
def test_rejection_capped_bit_exact(dt):
    w = _w(1 << 16, dt, 8)
    cap = float(np.median(w))
    a, out_w, trips = pf.rejection_ancestors_capped(w, cap, pf.RngStream(1005, (4,)), return_trips=True,
                                                    rng_mode="numpy")
    a_ref, trips_ref, w_ref = O.rejection_stream(w, 0.0, 1005, (4,), cap=cap)
    np.testing.assert_array_equal(np_(a), a_ref)
    np.testing.assert_array_equal(np_(trips), trips_ref)
    np.testing.assert_array_equal(np_(out_w), w_ref)


@pytest.mark.parametrize("case", [c[0] for c in WEIGHT_CASES if c[1] <= 5000])
def test_rejection_golden(golden, case):
    """The reference's own outputs (golden), including non-power-of-two N
    (Lemire redraws possible) and exact zeros."""
    nm, n, seed, sigma, dtype, zeros = next(c for c in WEIGHT_CASES if c[0] == case)
    w = golden_weights(n, seed, sigma, dtype, zeros)
    rs = pf.RngStream(1000 + seed, (3, 5))
    a, trips = pf.rejection_ancestors(w, float(w.max()), rs, return_trips=True, rng_mode="numpy")
    np.testing.assert_array_equal(np_(a), golden[f"{case}/rej_a"])
    np.testing.assert_array_equal(np_(trips), golden[f"{case}/rej_trips"])
    cap = float(np.median(w))
    a, out_w, trips = pf.rejection_ancestors_capped(w, cap, rs, return_trips=True, rng_mode="numpy")
    np.testing.assert_array_equal(np_(a), golden[f"{case}/cap_a"])
    np.testing.assert_array_equal(np_(out_w), golden[f"{case}/cap_w"])
    np.testing.assert_array_equal(np_(trips), golden[f"{case}/cap_trips"])


@pytest.mark.parametrize("case", [c[0] for c in WEIGHT_CASES if c[1] <= 5000])
@pytest.mark.parametrize("alg", ["multinomial", "stratified", "systematic", "rejection", "rejection-capped"])
def test_delivery_golden_serial(golden, case, alg):
    """Every delivery through the facade equals the reference's (golden), f32
    cases included, with accum='serial'."""
    nm, n, seed, sigma, dtype, zeros = next(c for c in WEIGHT_CASES if c[0] == case)
    w = golden_weights(n, seed, sigma, dtype, zeros)
    cfg = pf.ResamplerConfig(alg, b=32, sup_w=float(w.max()), sup_v=float(np.median(w)))
    kw = {"accum": "serial"} if alg in ("multinomial", "stratified", "systematic") else {}
    c = np_(pf.deliver(w, cfg, pf.RngStream(2000 + seed, (7,)), rng_mode="numpy", **kw))
    np.testing.assert_array_equal(c, golden[f"{case}/deliver/{alg}"])


# ---------------------------------------------------------------------------
# the C2 delivery workload end to end: 5 resamplers x f32/f64 at 2^20


@pytest.mark.parametrize("dt", list(DT))
@pytest.mark.parametrize("alg", ["multinomial", "stratified", "systematic", "metropolis", "rejection"])
def test_c2_delivery_bit_exact(c2, dt, alg):
    """resample_ancestors + permute_parallel (the reference's timed region,
    bench.py:155-161) at N = 2^20, element by element."""
    w = c2[dt]
    cfg = pf.ResamplerConfig(alg, b=32)
    kw = {"accum": "serial"} if alg in ("multinomial", "stratified", "systematic") else {}
    c = np_(pf.deliver(w, cfg, pf.RngStream(3000, (11,)), rng_mode="numpy", **kw))
    np.testing.assert_array_equal(c, O.deliver(w, alg, 3000, (11,), b=32))


# ---------------------------------------------------------------------------
# default accumulation (accum="f64"): the fast path


@pytest.mark.parametrize("alg", ["systematic", "stratified"])
def test_c2_default_f64_bit_exact(c2, alg):
    """float64 weights, the parallel float64 scan: no rounding-fragile
    position at 2^20, so O and the delivery equal the reference."""
    w = c2["f64"]
    rs = pf.RngStream(1006, (1,))
    if alg == "systematic":
        got = np_(pf.systematic_cumulative_offspring(w, rs, rng_mode="numpy"))
        want = O.systematic(w, O.systematic_offset(1006, (1,)))
    else:
        got = np_(pf.stratified_cumulative_offspring(w, rs, rng_mode="numpy"))
        want = O.stratified(w, O.stratified_uniforms(1006, (1,), w.size))
    assert np.flatnonzero(got != want).size == 0
    c = np_(pf.deliver(w, pf.ResamplerConfig(alg), rs, rng_mode="numpy"))
    np.testing.assert_array_equal(c, O.permute(O.expand_cumulative(want)))


def test_c2_default_f64_multinomial_bit_exact(c2):
    w = c2["f64"]
    a = np_(pf.multinomial_ancestors(w, pf.RngStream(1007), rng_mode="numpy"))
    np.testing.assert_array_equal(a, O.multinomial_stream(w, 1007, ()))


def _f64_fold_positions(w32, u):
    """O from a float64 fold of the float32 weights with the float32-rounded
    offset widened (what accum='f64' computes, up to reassociation)."""
    n = w32.size
    W = np.cumsum(w32.astype(np.float64))
    r = W * float(n) / W[-1]
    O_ = np.minimum(np.floor(r + np.float64(np.float32(u))), n).astype(np.int64)
    O_ = np.maximum.accumulate(O_)
    O_[-1] = n
    return O_


@pytest.mark.parametrize("n_log2", [20, 24])
def test_f32_systematic_tolerance_vs_reference(n_log2):
    """Stated float32 tolerance.  The reference folds float32
    serially (its W drifts: SURVEY A.4); the default path carries float64.
    Asserted: (1) accum='serial' equals the reference's float32 output
    exactly; (2) the default output is within 1 position of the float64 fold
    of the same float32 weights; (3) hence its distance to the reference's
    output is at most the reference's own drift + 1; (4) per-parent
    |o - N w/sum w| < 1 (systematic's bound)."""
    n = 1 << n_log2
    w = _w(n, "f32", 40 + n_log2)
    rs = pf.RngStream(1008, (n_log2,))
    u = O.systematic_offset(1008, (n_log2,))
    O_ref = O.systematic(w, u).astype(np.int64)
    O_ser = np_(pf.systematic_cumulative_offspring(w, rs, rng_mode="numpy", accum="serial")).astype(np.int64)
    np.testing.assert_array_equal(O_ser, O_ref)
    O_gpu = np_(pf.systematic_cumulative_offspring(w, rs, rng_mode="numpy")).astype(np.int64)
    O_64 = _f64_fold_positions(w, u)
    assert np.abs(O_gpu - O_64).max() <= 1
    drift_ref = np.abs(O_ref - O_64).max()
    assert np.abs(O_gpu - O_ref).max() <= drift_ref + 1
    o = np.diff(O_gpu, prepend=0)
    m = w.astype(np.float64) * n / w.astype(np.float64).sum()
    assert np.abs(o - m).max() < 1 + 1e-6
    print(f"2^{n_log2} f32: reference drift max|O_ref - O_f64| = {drift_ref}, "
          f"max|O_gpu - O_ref| = {np.abs(O_gpu - O_ref).max()}, max|O_gpu - O_f64| = {np.abs(O_gpu - O_64).max()}")
