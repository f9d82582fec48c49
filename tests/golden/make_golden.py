"""Generate golden vectors by running the REFERENCE implementation.

Run in the development container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``pfresample`` read-only from /root/reference/pkg/src, evaluates
the hot-path functions on seeded inputs and writes ``tests/golden/golden.npz``
(committed).  Nothing at test/bench time reads /root/reference: the fixtures
travel with the repository.

Weights are regenerated in the tests from the recorded seeds with
``golden_weights`` below (numpy PCG64 + ziggurat normals, identical on the GPU
box which runs the same image); a float64 checksum of each weight vector is
stored so a generator drift would be detected rather than silently accepted.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


def golden_weights(n: int, seed: int, sigma: float = 1.0, dtype=np.float64, zeros: float = 0.0):
    """i.i.d. log-normal weights w = exp(lw - max lw), lw ~ N(0, sigma^2);
    optionally a fraction of exact zeros."""
    g = np.random.default_rng(seed)
    lw = g.normal(0.0, sigma, n)
    w = np.exp(lw - lw.max())
    if zeros:
        w[g.random(n) < zeros] = 0.0
        if not (w > 0).any():
            w[0] = 1.0
    return w.astype(dtype)


def golden_ancestry(n: int, seed: int, sorted_: bool = False):
    g = np.random.default_rng(seed)
    a = g.integers(0, n, size=n)
    return np.sort(a) if sorted_ else a


# (name, n, seed, sigma, dtype, zeros)
WEIGHT_CASES = [
    ("w1000_f64", 1000, 11, 1.0, np.float64, 0.0),
    ("w1000_f32", 1000, 12, 1.0, np.float32, 0.0),
    ("w1024_f64", 1024, 13, 1.0, np.float64, 0.0),
    ("w1024_f32", 1024, 14, 1.0, np.float32, 0.0),
    ("w777z_f64", 777, 15, 2.0, np.float64, 0.3),
    ("w4096_f32", 4096, 16, 0.5, np.float32, 0.0),
    ("w65536_f64", 1 << 16, 17, 1.0, np.float64, 0.0),  # BASELINE config 1
]

ANCESTRY_CASES = [(1, 21), (2, 22), (3, 23), (7, 24), (100, 25), (257, 26), (4096, 27)]

# (n, dtype) of the stable_sum fixtures; vectors regenerated from their index
STABLE_CASES = [(1, np.float64), (5, np.float32), (4096, np.float64), (4097, np.float32), (100000, np.float64),
                (1 << 20, np.float32)]


def stable_vector(k: int) -> np.ndarray:
    n, dt = STABLE_CASES[k]
    g = np.random.default_rng(600 + k)
    return (g.random(n) * np.exp(g.normal(0, 4, n))).astype(dt)


def main():
    sys.path.insert(0, REF_SRC)
    import pfresample as pf
    from pfresample import ancestry as anc

    out = {}

    for name, n, seed, sigma, dtype, zeros in WEIGHT_CASES:
        w = golden_weights(n, seed, sigma, dtype, zeros)
        out[f"{name}/checksum"] = np.float64(w.astype(np.float64).sum())
        if n <= 5000:
            out[f"{name}/W"] = pf.inclusive_prefix_sum(w)
            out[f"{name}/Wex"] = pf.exclusive_prefix_sum(w)
        rs = pf.RngStream(1000 + seed, (3, 5))
        O_sys = pf.systematic_cumulative_offspring(w, rs)
        out[f"{name}/sys_O"] = O_sys.astype(np.int32)
        a_sys = pf.cumulative_offspring_to_ancestors(O_sys)
        c_sys, steps = pf.permute_parallel(a_sys, return_max_steps=True)
        out[f"{name}/sys_c"] = c_sys.astype(np.int32)
        out[f"{name}/sys_steps"] = np.int64(steps)
        if n > 5000:
            continue
        out[f"{name}/str_O"] = pf.stratified_cumulative_offspring(w, rs).astype(np.int32)
        out[f"{name}/mult_a"] = pf.multinomial_ancestors(w, rs).astype(np.int32)
        out[f"{name}/mser_a"] = pf.multinomial_ancestors_serial(w, rs).astype(np.int32)
        out[f"{name}/metro_a"] = pf.metropolis_ancestors(w, 32, rs).astype(np.int32)
        a_rej, trips = pf.rejection_ancestors(w, float(w.max()), rs, return_trips=True)
        out[f"{name}/rej_a"] = a_rej.astype(np.int32)
        out[f"{name}/rej_trips"] = trips.astype(np.int32)
        cap = float(np.median(w))
        a_cap, w_cap, trips_cap = pf.rejection_ancestors_capped(w, cap, rs, return_trips=True)
        out[f"{name}/cap_a"] = a_cap.astype(np.int32)
        out[f"{name}/cap_w"] = w_cap
        out[f"{name}/cap_trips"] = trips_cap.astype(np.int32)
        # the full delivery for every algorithm through the reference facade
        for alg in pf.ALGORITHMS:
            cfg = pf.ResamplerConfig(algorithm=alg, b=32, sup_w=float(w.max()), sup_v=cap)
            res = pf.resample_ancestors(w, cfg, pf.RngStream(2000 + seed, (7,)))
            out[f"{name}/deliver/{alg}"] = anc.permute_parallel(res.ancestors).astype(np.int32)

    for n, seed in ANCESTRY_CASES:
        for sorted_ in (False, True):
            a = golden_ancestry(n, seed, sorted_)
            tag = f"anc{n}_{'s' if sorted_ else 'u'}"
            out[f"{tag}/d"] = pf.prepermute(a).astype(np.int32)
            c, steps = pf.permute_parallel(a, return_max_steps=True)
            out[f"{tag}/c"] = c.astype(np.int32)
            out[f"{tag}/steps"] = np.int64(steps)
            out[f"{tag}/serial"] = pf.permute_serial(a).astype(np.int32)
            o = pf.ancestors_to_offspring(a)
            out[f"{tag}/o"] = o.astype(np.int32)
            O = pf.offspring_to_cumulative(o)
            out[f"{tag}/O"] = O.astype(np.int32)
            out[f"{tag}/expand"] = pf.cumulative_offspring_to_ancestors(O).astype(np.int32)

    # log-weights adapter
    g = np.random.default_rng(31)
    lw = g.normal(0, 3, 500)
    lw[::17] = -np.inf
    out["logw/lw"] = lw
    out["logw/w"] = pf.logweights_to_weights(lw)
    out["logw/w32"] = pf.logweights_to_weights(lw.astype(np.float32))

    # Metropolis step recipe
    grid = [(0.5, 0.005, 16), (1.0, 0.01, 4), (0.05, None, 1 << 10), (1e-3, None, 1 << 16), (0.3, 0.1, 64)]
    out["msteps/args"] = np.array([[p, -1.0 if e is None else e, n] for p, e, n in grid])
    out["msteps/B"] = np.array([pf.metropolis_num_steps(p, e, n) for p, e, n in grid], dtype=np.int64)

    # Reference-stream layout: raw draws a Metropolis call consumes
    rs = pf.RngStream(4242, (1, 2, 3))
    gen = rs.generator()
    out["stream/u"] = gen.random(64)
    out["stream/j1024"] = gen.integers(0, 1024, size=64)
    out["stream/j1000"] = gen.integers(0, 1000, size=65)
    out["stream/u2"] = gen.random(8)
    out["stream/derive"] = np.array([pf.derive_seed(4242, 0, 1, 2, 3), pf.derive_seed(4242, 1, 1, 2, 3),
                                     pf.derive_seed(0), pf.derive_seed(2**64 - 1, 5)], dtype=np.uint64)

    # stable_sum (pairwise tree), ESS and resampling MSE (diagnostics.py:54-80)
    for k, (n, dt) in enumerate(STABLE_CASES):
        v = stable_vector(k)
        out[f"stable/{k}/checksum"] = np.float64(v.astype(np.float64).sum())
        out[f"stable/{k}/sum"] = np.asarray(pf.stable_sum(v))
    for k, n in enumerate((16, 1000, 4097)):
        g = np.random.default_rng(700 + k)
        w = np.exp(g.normal(0, 1, n))
        o = np.bincount(g.integers(0, n, n), minlength=n)
        out[f"wstats/{k}/w"] = w
        out[f"wstats/{k}/o"] = o.astype(np.int64)
        out[f"wstats/{k}/ess"] = np.float64(pf.ess(w))
        out[f"wstats/{k}/mse"] = np.float64(pf.resampling_mse(o, w))

    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {len(out)} arrays to {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
