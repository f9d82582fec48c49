"""CPU oracle for the resampling hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference package ``pfresample``
(``/root/reference/pkg/src/pfresample``) for the functions on the hot path
listed in SURVEY.md section 8(a).  It exists so that

* the parity tests under ``tests/`` can check the CUDA path element by element,
* ``__graft_entry__.smoke()`` can check one small GPU invocation, and
* ``bench.py`` can time the reference algorithm on the host cores
  (``cpu_baseline`` / ``--impl reference``).

Nothing in the product package (``paper_1301_4019_b200``) imports it: the
product path runs on the GPU or raises.

Parity pinning: the restatement is checked against golden vectors produced by
the reference itself (``tests/golden/make_golden.py`` imports the read-only
reference and writes ``tests/golden/*.npz``) and against the reference's own
known-answer tests (restated in ``tests/test_oracle.py``).

Every function cites the reference ``file:line`` it restates; the paths are
relative to ``/root/reference/pkg/src/pfresample``.
"""

from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1

# ---------------------------------------------------------------------------
# RNG addressing (rng.py:22-74)

_SPLITMIX_GAMMA = 0x9E3779B97F4A7C15
_SPLITMIX_M1 = 0xBF58476D1CE4E5B9
_SPLITMIX_M2 = 0x94D049BB133111EB


def _finalise64(z: int) -> int:
    """splitmix64 output function (rng.py:28-32)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * _SPLITMIX_M1) & MASK64
    z = ((z ^ (z >> 27)) * _SPLITMIX_M2) & MASK64
    return z ^ (z >> 31)


def derive_seed(seed: int, *ids: int) -> int:
    """Key derivation of rng.py:39-49: absorb len(ids) then each id."""
    h = _finalise64(int(seed))
    for v in (len(ids),) + tuple(int(i) for i in ids):
        h = _finalise64((h + _SPLITMIX_GAMMA + (v & MASK64)) & MASK64)
    return h


def stream_key(seed: int, ids=()) -> tuple[int, int]:
    """The Philox4x64 key numpy is seeded with in RngStream.generator (rng.py:69-74)."""
    ids = tuple(int(i) for i in ids)
    return derive_seed(seed, 0, *ids), derive_seed(seed, 1, *ids)


def generator(seed: int, ids=()) -> np.random.Generator:
    """numpy Generator positioned at the start of stream (seed, ids) (rng.py:69-74)."""
    k0, k1 = stream_key(seed, ids)
    return np.random.Generator(np.random.Philox(key=np.array([k0, k1], dtype=np.uint64)))


# Philox4x64-10 in pure Python (Salmon et al. 2011, the generator numpy wraps).
_PH64_M = (0xD2E7470EE14C6C93, 0xCA5A826395121157)
_PH64_W = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)


def philox4x64_10(counter, key):
    """One Philox4x64-10 block; numpy's k-th raw u64 is block(k//4 + 1)[k % 4]."""
    x = [int(c) & MASK64 for c in counter]
    k0, k1 = int(key[0]) & MASK64, int(key[1]) & MASK64
    for rnd in range(10):
        if rnd:
            k0 = (k0 + _PH64_W[0]) & MASK64
            k1 = (k1 + _PH64_W[1]) & MASK64
        p0 = _PH64_M[0] * x[0]
        p1 = _PH64_M[1] * x[2]
        x = [(p1 >> 64) ^ x[1] ^ k0, p1 & MASK64, (p0 >> 64) ^ x[3] ^ k1, p0 & MASK64]
    return x


_PH32_M = (0xD2511F53, 0xCD9E8D57)
_PH32_W = (0x9E3779B9, 0xBB67AE85)
MASK32 = 0xFFFFFFFF


def philox4x32_10(counter, key):
    """Philox4x32-10 block (the GPU's own generator, see csrc/pfr_rng.cuh)."""
    x = [int(c) & MASK32 for c in counter]
    k0, k1 = int(key[0]) & MASK32, int(key[1]) & MASK32
    for rnd in range(10):
        if rnd:
            k0 = (k0 + _PH32_W[0]) & MASK32
            k1 = (k1 + _PH32_W[1]) & MASK32
        p0 = _PH32_M[0] * x[0]
        p1 = _PH32_M[1] * x[2]
        x = [(p1 >> 32) ^ x[1] ^ k0, p1 & MASK32, (p0 >> 32) ^ x[3] ^ k1, p0 & MASK32]
    return x


# ---------------------------------------------------------------------------
# weight validation (diagnostics.py:38-51, 138-155; primitives.py:23-31)


def as_weights(w, require_positive_total: bool = True) -> np.ndarray:
    """check_weights (diagnostics.py:38-51)."""
    v = np.asarray(w)
    if v.ndim != 1 or v.size == 0:
        raise ValueError("w must be a one-dimensional vector with at least one element")
    if not np.issubdtype(v.dtype, np.floating):
        v = v.astype(np.float64)
    if not np.isfinite(v).all():
        raise ValueError("w must be finite (no NaN or infinity)")
    if v.min() < 0:
        raise ValueError("w must be non-negative")
    if require_positive_total and not (v > 0).any():
        raise ValueError("w must contain at least one strictly positive weight")
    return v


def logweights_to_weights(lw) -> np.ndarray:
    """Max-shift then exp (diagnostics.py:138-155)."""
    v = np.asarray(lw)
    if v.ndim != 1 or v.size == 0:
        raise ValueError("log-weight vector must be one-dimensional and non-empty")
    if not np.issubdtype(v.dtype, np.floating):
        v = v.astype(np.float64)
    if np.isnan(v).any() or (v == np.inf).any():
        raise ValueError("log-weights may not contain NaN or +inf")
    top = v.max()
    if top == -np.inf:
        raise ValueError("all log-weights are -inf: no positive weight")
    return np.exp(v - top)


# ---------------------------------------------------------------------------
# primitives (primitives.py:34-106)


def inclusive_scan(w) -> np.ndarray:
    """Strict left fold in the input precision (primitives.py:34-42)."""
    return np.cumsum(np.asarray(w))


def exclusive_scan(w) -> np.ndarray:
    """Shifted fold with leading zero (primitives.py:45-51)."""
    w = np.asarray(w)
    out = np.zeros_like(w)
    if w.size > 1:
        out[1:] = np.cumsum(w[:-1])
    return out


def stable_sum(w):
    """Balanced pairwise tree over the zero-padded power-of-two vector
    (primitives.py:69-88)."""
    w = np.asarray(w)
    n = w.size
    size = 1 << (n - 1).bit_length()
    v = np.zeros(size, dtype=w.dtype)
    v[:n] = w
    while v.size > 1:
        v = v[0::2] + v[1::2]
    return v[0]


def ess(w) -> float:
    """(sum w)^2 / (w . w) (diagnostics.py:54-63)."""
    w = as_weights(w)
    total = w.sum(dtype=w.dtype)
    return float(total * total / np.dot(w, w))


def resampling_mse(o, w) -> float:
    """(1/N) sum (o/N - w/sum w)^2 in float64 (diagnostics.py:66-80)."""
    o = np.asarray(o, dtype=np.float64)
    w = as_weights(w).astype(np.float64)
    diff = o / w.size - w / w.sum()
    return float(np.mean(diff * diff))


def adjacent_difference(W) -> np.ndarray:
    """primitives.py:54-57."""
    W = np.asarray(W)
    out = W.copy()
    out[1:] = W[1:] - W[:-1]
    return out


def lower_bound(W, u) -> np.ndarray:
    """searchsorted(side='left') clamped to N-1 (primitives.py:91-106).

    Mixed precision: numpy promotes a float32 W against float64 queries to
    float64 before comparing."""
    W = np.asarray(W)
    idx = np.searchsorted(W, u, side="left")
    return np.minimum(idx, W.size - 1)


# ---------------------------------------------------------------------------
# resamplers (resamplers.py)


def offspring_from_positions(w: np.ndarray, u_per_stratum: np.ndarray) -> np.ndarray:
    """Cumulative offspring from strata offsets (resamplers.py:139-153).

    All arithmetic in w's precision: r = W*N/W[-1] (multiply, then divide),
    1-based stratum k = min(N, floor(r)+1), O = min(N, floor(r + u[k-1])),
    then the monotone repair and O[-1] = N."""
    n = w.size
    t = w.dtype.type
    W = np.cumsum(w)
    r = (W * t(n)) / W[-1]
    stratum = np.minimum(n, np.floor(r).astype(np.int64) + 1)
    O = np.floor(r + u_per_stratum[stratum - 1]).astype(np.int64)
    O = np.minimum(O, n)
    O = np.maximum.accumulate(O)
    O[-1] = n
    return O


def systematic_offset(seed: int, ids=()) -> float:
    """The single draw systematic resampling takes (resamplers.py:134)."""
    return float(generator(seed, ids).random())


def systematic(w, offset: float) -> np.ndarray:
    """resamplers.py:127-136 with an explicit offset."""
    w = as_weights(w)
    return offspring_from_positions(w, np.full(w.size, offset, dtype=w.dtype))


def stratified(w, uniforms) -> np.ndarray:
    """resamplers.py:105-124 with explicit per-stratum uniforms (cast to w's dtype)."""
    w = as_weights(w)
    u = np.asarray(uniforms, dtype=np.float64).astype(w.dtype)
    return offspring_from_positions(w, u)


def stratified_uniforms(seed: int, ids, n: int) -> np.ndarray:
    return generator(seed, ids).random(n)


def multinomial(w, scaled_uniforms) -> np.ndarray:
    """resamplers.py:56-74 with injected pre-scaled draws in [0, W[-1])."""
    w = as_weights(w)
    W = np.cumsum(w)
    return lower_bound(W, np.asarray(scaled_uniforms, dtype=np.float64)).astype(np.int64)


def multinomial_stream(w, seed: int, ids=()) -> np.ndarray:
    """resamplers.py:66-69: u = random(N) * float(W[-1])."""
    w = as_weights(w)
    total = float(np.cumsum(w)[-1])
    u = generator(seed, ids).random(w.size) * total
    return multinomial(w, u)


def multinomial_sorted(w, seed: int, ids=()) -> np.ndarray:
    """Sorted order statistics by log spacings, descending sweep (resamplers.py:77-102)."""
    w = as_weights(w)
    n = w.size
    Wx = exclusive_scan(w).tolist()
    total = float(Wx[-1]) + float(w[-1])
    draws = generator(seed, ids).random(n)
    out = np.empty(n, dtype=np.int64)
    log_top = 0.0
    j = n - 1
    for pos in range(n):
        i = n - 1 - pos
        d = draws[pos]
        log_top += (math.log(d) if d > 0.0 else -math.inf) / (i + 1)
        target = total * math.exp(log_top)
        while target < Wx[j]:
            j -= 1
        out[i] = j
    return out


def metropolis_steps(p_star: float, epsilon, n: int) -> int:
    """Two-state bias bound (resamplers.py:168-201)."""
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
        raise ValueError(f"bias bound invalid: lambda = {lam} <= 0 (p_star too small relative to N={n})")
    b = math.log(eps * (alpha + beta) / max(alpha, beta)) / math.log(lam)
    return max(1, math.floor(b) + 1)


def metropolis_draws(seed: int, ids, n: int, steps: int):
    """The (u, j) sequence metropolis_ancestors consumes (resamplers.py:223-227):
    per step N float64 uniforms, then N integers in [0, N), from one generator."""
    g = generator(seed, ids)
    us = np.empty((steps, n))
    js = np.empty((steps, n), dtype=np.int64)
    for b in range(steps):
        us[b] = g.random(n)
        js[b] = g.integers(0, n, size=n)
    return us, js


def metropolis_replay(w, us, js) -> np.ndarray:
    """Chains started at their own index; accept iff w[k]==0 or u <= w[j]/w[k]
    with the ratio rounded in w's dtype and compared in float64
    (resamplers.py:224-234; erratum k <- j)."""
    w = as_weights(w, require_positive_total=False)
    k = np.arange(w.size, dtype=np.int64)
    for u, j in zip(us, js):
        wk = w[k]
        with np.errstate(divide="ignore", invalid="ignore"):
            ratio = w[j] / wk
        move = (wk == 0) | (u <= ratio)
        k = np.where(move, j, k)
    return k


def metropolis_stream(w, steps: int, seed: int, ids=()) -> np.ndarray:
    """metropolis_ancestors (resamplers.py:204-234) with the draws taken step by
    step from the generator, as the reference does (no (B, N) draw arrays)."""
    w = as_weights(w, require_positive_total=False)
    n = w.size
    g = generator(seed, ids)
    k = np.arange(n, dtype=np.int64)
    for _ in range(int(steps)):
        u = g.random(n)
        j = g.integers(0, n, size=n)
        wk = w[k]
        with np.errstate(divide="ignore", invalid="ignore"):
            ratio = w[j] / wk
        k = np.where((wk == 0) | (u <= ratio), j, k)
    return k


class StreamModel:
    """numpy's Generator(Philox) as the resamplers consume it, restated from
    the raw Philox4x64-10 words (numpy distributions.c / philox.h): random()
    takes one fresh u64 ((x >> 11) 2^-53); integers(0, N) takes 32-bit words
    from next_uint32 -- the LOW half of a fresh u64, the high half buffered
    for the next 32-bit request (the buffer survives across calls; random()
    never touches it) -- mapped by Lemire's method, (u32 * N) >> 32, redrawn
    while the low product word is below (2^32 - N) mod N.  Pure Python: small
    draws only (pinned by the golden stream vectors)."""

    def __init__(self, seed: int, ids=()):
        self.key = stream_key(seed, ids)
        self.q = 0
        self.buf = None

    def _word(self, k: int) -> int:
        return philox4x64_10([k // 4 + 1, 0, 0, 0], self.key)[k % 4]

    def random(self, m: int) -> np.ndarray:
        out = [(self._word(self.q + i) >> 11) * 2.0**-53 for i in range(m)]
        self.q += m
        return np.array(out)

    def _u32(self) -> int:
        if self.buf is not None:
            v, self.buf = self.buf, None
            return v
        x = self._word(self.q)
        self.q += 1
        self.buf = x >> 32
        return x & 0xFFFFFFFF

    def integers(self, n: int, m: int) -> np.ndarray:
        thr = ((1 << 32) - n) % n
        out = []
        for _ in range(m):
            while True:
                p = self._u32() * n
                if (p & 0xFFFFFFFF) >= thr:
                    break
            out.append(p >> 32)
        return np.array(out, dtype=np.int64)


def rejection_stream(w, bound: float, seed: int, ids=(), cap=None):
    """Round-synchronous rejection loop (resamplers.py:237-310).

    Slot i first proposes itself; pending slots then draw, per round, one
    integer each and one uniform each (integers for the whole pending set
    first, then uniforms), accepting when beta <= v[j]/bound.  ``cap`` gives
    the capped variant (resamplers.py:258-279): v = min(w, cap), returned
    importance weights w[a]/v[a] (1 where v[a]==0).  Returns (a, trips[, out_w])."""
    w = as_weights(w, require_positive_total=False)
    bound = float(bound if cap is None else cap)
    if not math.isfinite(bound) or bound <= 0:
        raise ValueError(f"weight bound must be finite and positive, got {bound}")
    v = w if cap is None else np.minimum(w, w.dtype.type(cap))
    n = v.size
    ratio = v / v.dtype.type(bound)
    if not np.isfinite(ratio).all():
        raise ValueError("non-finite acceptance ratio: weight bound underflows the weights")
    g = generator(seed, ids)
    a = np.arange(n, dtype=np.int64)
    trips = np.ones(n, dtype=np.int64)
    pending = np.flatnonzero(g.random(n) > ratio)
    rounds = 0
    while pending.size:
        rounds += 1
        if rounds > 100_000:
            raise RuntimeError("rejection resampling made no progress after 100000 rounds")
        j = g.integers(0, n, size=pending.size)
        beta = g.random(pending.size)
        ok = beta <= ratio[j]
        a[pending[ok]] = j[ok]
        trips[pending] += 1
        pending = pending[~ok]
    if cap is None:
        return a, trips
    with np.errstate(invalid="ignore", divide="ignore"):
        out_w = w[a] / v[a]
    out_w = np.where(v[a] == 0, w.dtype.type(1), out_w).astype(w.dtype)
    return a, trips, out_w


# ---------------------------------------------------------------------------
# the GPU's own Philox stream (rng_mode='philox'): a model of its rejection


def philox4x32_10_vec(c0, c1, c2, c3, k0: int, k1: int):
    """philox4x32_10 over numpy arrays of 32-bit counters (uint64 lanes)."""
    x0, x1, x2, x3 = (np.asarray(c, dtype=np.uint64) & MASK32 for c in (c0, c1, c2, c3))
    x0, x1, x2, x3 = (np.broadcast_to(v, np.broadcast(x0, x1, x2, x3).shape).copy() for v in (x0, x1, x2, x3))
    m0, m1 = np.uint64(_PH32_M[0]), np.uint64(_PH32_M[1])
    sh, lo = np.uint64(32), np.uint64(MASK32)
    for rnd in range(10):
        if rnd:
            k0 = (k0 + _PH32_W[0]) & MASK32
            k1 = (k1 + _PH32_W[1]) & MASK32
        p0 = m0 * x0  # < 2^64: no wrap
        p1 = m1 * x2
        x0, x1, x2, x3 = ((p1 >> sh) ^ x1 ^ np.uint64(k0), p1 & lo, (p0 >> sh) ^ x3 ^ np.uint64(k1), p0 & lo)
    return x0, x1, x2, x3


TAG_REJECTION = 0x524A  # csrc/pfr_rng.cuh kTagRejection


def own_rejection(w, bound: float, key0: int, cap=None):
    """The GPU's own-stream rejection (csrc/pfr_resample.cu rej_draws,
    k_rejection_philox) for a power-of-two N: trip t of slot i uses Philox
    counter (i, t // 2, tag, 0) keyed (key0 low, key0 high), words 2(t&1) /
    2(t&1)+1 = proposal (umulhi(x, N)) / open uniform; trip 0 proposes i;
    accept when beta * bound <= v[j] in the weights' precision (the
    semantics of resamplers.py:237-310 on this stream).  Returns (a, trips[,
    out_w]).  Test model of the product's stream, not of the reference's."""
    w = np.asarray(w)
    n = w.size
    if n & (n - 1):
        raise ValueError("the model covers power-of-two N (no Lemire redraws)")
    T = w.dtype.type
    capv = T(cap) if cap is not None else None
    v = w if cap is None else np.where(w < capv, w, capv)
    bnd = T(cap if cap is not None else bound)
    k0, k1 = int(key0) & MASK32, (int(key0) >> 32) & MASK32
    a = np.full(n, -1, dtype=np.int64)
    trips = np.zeros(n, dtype=np.int64)
    active = np.arange(n, dtype=np.int64)
    t = 0
    while active.size:
        if t > 1 << 20:
            raise RuntimeError("no progress")
        o = philox4x32_10_vec(active, t // 2, TAG_REJECTION, 0, k0, k1)
        for h in (0, 1):
            if not active.size:
                break
            if len(o[0]) != active.size:  # slots accepted on the first half
                o = tuple(x[keep] for x in o)
            xj, xu = o[2 * h], o[2 * h + 1]
            j = ((xj * np.uint64(n)) >> np.uint64(32)).astype(np.int64)
            if t == 0:
                j = active.copy()
            if T is np.float32:
                u = ((((xu >> np.uint64(9)) << np.uint64(1)) | np.uint64(1)).astype(np.float32)
                     * np.float32(1.0 / 16777216.0))
            else:
                u = xu.astype(np.float64) * 2.0 ** -32 + 2.0 ** -33
            ok = u * bnd <= v[j]
            a[active[ok]] = j[ok]
            trips[active[ok]] = t + 1
            keep = ~ok
            active = active[keep]
            t += 1
        if t % 2:  # odd: the loop broke after the first half
            t += 1
    if cap is None:
        return a, trips
    va = v[a]
    with np.errstate(invalid="ignore", divide="ignore"):
        out_w = np.where(va == 0, T(1), w[a] / va).astype(w.dtype)
    return a, trips, out_w


# ---------------------------------------------------------------------------
# ancestry (ancestry.py)


def expand_cumulative(O) -> np.ndarray:
    """Parent v fills slots [O[v-1], O[v]) (ancestry.py:69-76)."""
    O = np.asarray(O, dtype=np.int64)
    counts = np.diff(O, prepend=0)
    return np.repeat(np.arange(O.size, dtype=np.int64), counts)


def histogram(a) -> np.ndarray:
    """ancestry.py:79-82."""
    a = np.asarray(a, dtype=np.int64)
    return np.bincount(a, minlength=a.size).astype(np.int64)


def prepermute(a) -> np.ndarray:
    """d[v] = lowest slot whose parent is v, sentinel N (ancestry.py:125-136)."""
    a = np.asarray(a, dtype=np.int64)
    n = a.size
    d = np.full(n, n, dtype=np.int64)
    # first occurrence of each value: reversed assignment leaves the lowest index
    d[a[::-1]] = np.arange(n - 1, -1, -1, dtype=np.int64)
    return d


def permute(a, with_steps: bool = False):
    """Claim-and-chase permutation (ancestry.py:139-174).

    Losers (slots whose claim lost) follow x <- d[x] to a sentinel slot and
    claim it; ascending loser order, as the reference (the outcome does not
    depend on the order: SURVEY.md finding 3).  c = a[d]."""
    a = np.asarray(a, dtype=np.int64)
    n = a.size
    d = prepermute(a)
    losers = np.flatnonzero(d[a] != np.arange(n))
    dl = d.tolist()
    longest = 0
    for i in losers.tolist():
        x = i
        hops = 0
        while dl[x] != n:
            x = dl[x]
            hops += 1
            if hops > n:
                raise RuntimeError("permutation chain walk failed to terminate")
        dl[x] = i
        if hops > longest:
            longest = hops
    c = a[np.asarray(dl, dtype=np.int64)]
    return (c, longest) if with_steps else c


def permute_swaps(a) -> np.ndarray:
    """Serial pairwise swaps (ancestry.py:104-122)."""
    c = np.asarray(a, dtype=np.int64).tolist()
    i = 0
    n = len(c)
    while i < n:
        v = c[i]
        if v != i and c[v] != v:
            c[i], c[v] = c[v], v
        else:
            i += 1
    return np.asarray(c, dtype=np.int64)


def satisfies_predicate(c) -> bool:
    """o[i] > 0 => c[i] == i (ancestry.py:97-101)."""
    c = np.asarray(c, dtype=np.int64)
    used = np.flatnonzero(np.bincount(c, minlength=c.size) > 0)
    return bool((c[used] == used).all())


def deliver(w, algorithm: str, seed: int, ids=(), *, b=None, sup_w=None, sup_v=None):
    """The timed delivery of bench.py:155-161: resample_ancestors then
    permute_parallel (resamplers.py:362-397; ancestry.py:139-174)."""
    w = as_weights(w)
    if algorithm == "systematic":
        a = expand_cumulative(systematic(w, systematic_offset(seed, ids)))
    elif algorithm == "stratified":
        a = expand_cumulative(stratified(w, stratified_uniforms(seed, ids, w.size)))
    elif algorithm == "multinomial":
        a = multinomial_stream(w, seed, ids)
    elif algorithm == "multinomial-serial":
        a = multinomial_sorted(w, seed, ids)
    elif algorithm == "metropolis":
        a = metropolis_stream(w, 32 if b is None else b, seed, ids)
    elif algorithm == "rejection":
        a, _ = rejection_stream(w, float(w.max()) if sup_w is None else sup_w, seed, ids)
    elif algorithm == "rejection-capped":
        a, _, _ = rejection_stream(w, 0.0, seed, ids, cap=sup_v)
    else:
        raise ValueError(f"unknown algorithm {algorithm!r}")
    return permute(a)


# ---------------------------------------------------------------------------
# Exact Metropolis bias oracle: E[o] after B steps


def metropolis_expected_offspring(w, steps: int) -> np.ndarray:
    """1^T P^B for the independence sampler with uniform proposals, O(N) per
    step via sorted prefix sums; every chain starts at its own index."""
    w = np.asarray(w, dtype=np.float64)
    n = w.size
    order = np.argsort(w, kind="stable")
    ws = w[order]
    # r_j = sum_{k != j} min(1, w_k / w_j)
    below = np.concatenate(([0.0], np.cumsum(ws)))  # sum of smaller-or-equal (by rank)
    # ranks with ties grouped: for each j, count of elements with w >= w_j and sum of w < w_j
    lo = np.searchsorted(ws, ws, side="left")      # #elements with w < w_j
    sum_less = below[lo]
    count_geq = n - lo
    with np.errstate(divide="ignore", invalid="ignore"):
        r = (count_geq - 1) + np.where(ws > 0, sum_less / ws, 0.0)
    r = np.where(ws > 0, r, n - 1)  # zero-weight states always move
    v = np.ones(n)  # occupancy in sorted order
    hi = np.searchsorted(ws, ws, side="right")     # #elements with w <= w_j
    for _ in range(int(steps)):
        # inflow from k with w_k <= w_j (k != j): v_k / N each
        c_v = np.concatenate(([0.0], np.cumsum(v)))
        with np.errstate(divide="ignore", invalid="ignore"):
            vw = np.where(ws > 0, v / ws, 0.0)
        c_vw = np.concatenate(([0.0], np.cumsum(vw)))
        inflow_le = c_v[hi] - v
        # zero-weight sources always accept: include them regardless (they sit at the front)
        inflow_gt = ws * (c_vw[n] - c_vw[hi])
        newv = (inflow_le + inflow_gt) / n + v * (1.0 - r / n)
        # a zero-weight target is entered only from zero-weight states (whose
        # ratio is +inf), including by proposing itself: mass S0 / N
        zero_mass = v[ws == 0].sum()
        v = np.where(ws > 0, newv, zero_mass / n)
    out = np.empty(n)
    out[order] = v
    return out
