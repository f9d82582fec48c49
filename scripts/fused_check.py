"""Systematic/stratified delivery vs the unfused reference pipeline, on the GPU.

For each case: c = deliver(w) must equal permute_parallel(expand(O(w))) computed
from the same cumulative offspring (K1 + K2 storing O, the general expand and
the claim/walk permute) -- the in-place ancestry is unique given O.  Then
CUDA-event timings of the delivery at N=2^24 f32/f64 (L2 flushed)."""
import os
import sys
import time
import faulthandler

faulthandler.dump_traceback_later(90, exit=True)

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402

torch.cuda.set_device(0)


def weights(kind, n, dt, seed):
    g = np.random.default_rng(seed)
    if kind == "lognormal1":
        w = np.exp(g.normal(0, 1, n))
    elif kind == "lognormal3":
        w = np.exp(g.normal(0, 3, n))
    elif kind == "last":  # every slot owned by the last particle: extreme negative drift
        w = np.zeros(n)
        w[-1] = 1.0
    elif kind == "first":
        w = np.zeros(n)
        w[0] = 1.0
    elif kind == "ramp":  # weight grows along the vector: drift negative, then back
        w = np.linspace(0, 1, n) ** 4
    elif kind == "blocks":  # zero blocks of 3 tiles
        w = np.exp(g.normal(0, 1, n))
        w[(np.arange(n) // 12288) % 2 == 1] = 0.0
    else:
        raise ValueError(kind)
    if w.sum() == 0:
        w[-1] = 1.0
    return torch.from_numpy(w.astype(dt)).cuda()


def check(kind, n, dt, seed=1, stratified=False):
    w = weights(kind, n, dt, seed)
    cfg = pf.ResamplerConfig("stratified" if stratified else "systematic")
    rs = pf.RngStream(seed)
    c, ms = pf.deliver(w, cfg, rs, index_dtype=torch.int32, return_max_steps=True)
    fn = pf.stratified_cumulative_offspring if stratified else pf.systematic_cumulative_offspring
    O = fn(w, pf.RngStream(seed))
    a = pf.cumulative_offspring_to_ancestors(O)
    want, ms_want = pf.permute_parallel(a, return_max_steps=True)
    ok = torch.equal(c.long(), want.long()) and int(ms) == int(ms_want)
    if int(ms) != int(ms_want):
        print(f"max_steps {kind} n={n}: {int(ms)} vs {int(ms_want)}")
    bad = 0 if ok else int((c.long() != want.long()).sum())
    return ok, bad


fails = 0
cases = []
for n in (1, 2, 31, 4095, 4096, 4097, 12289, 65536 + 3, 1 << 20, (1 << 22) + 77):
    for kind in ("lognormal1", "lognormal3", "last", "first", "ramp", "blocks"):
        for dt in (np.float32, np.float64):
            cases.append((kind, n, dt, False))
cases += [("lognormal1", 1 << 24, np.float32, False), ("lognormal1", 1 << 24, np.float64, False),
          ("lognormal1", 1 << 20, np.float64, True), ("lognormal3", 1 << 22, np.float32, True)]
t0 = time.time()
for kind, n, dt, strat in cases:
    t1 = time.time()
    print(f"case {kind} n={n} {dt.__name__}", flush=True)
    ok, bad = check(kind, n, dt, stratified=strat)
    if time.time() - t1 > 2:
        print(f"slow case {kind} n={n} {dt.__name__}: {time.time() - t1:.1f} s", flush=True)
    if not ok:
        fails += 1
        print(f"MISMATCH {kind} n={n} {dt.__name__} strat={strat}: {bad} indices", flush=True)
print(f"{len(cases) - fails}/{len(cases)} cases identical ({time.time() - t0:.1f} s)", flush=True)

# repeated deliveries on one workspace (counters must reset) + concurrent streams
w = weights("lognormal1", 1 << 20, np.float32, 3)
ref = pf.deliver(w, pf.ResamplerConfig("systematic"), pf.RngStream(3), index_dtype=torch.int32)
for _ in range(20):
    again = pf.deliver(w, pf.ResamplerConfig("systematic"), pf.RngStream(3), index_dtype=torch.int32)
    assert torch.equal(again, ref)
streams = [torch.cuda.Stream() for _ in range(6)]
outs = []
for s in streams:
    with torch.cuda.stream(s):
        outs.append(pf.deliver(w, pf.ResamplerConfig("systematic"), pf.RngStream(3), index_dtype=torch.int32))
torch.cuda.synchronize()
assert all(torch.equal(o, ref) for o in outs)
print("repeat + concurrent streams: identical", flush=True)

pf.config.check = False
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for dt in (np.float32, np.float64):
    n = 1 << 24
    w = weights("lognormal1", n, dt, 1)
    c = torch.empty(n, dtype=torch.int32, device="cuda")
    ts = []
    for r in range(20):
        flush.zero_()
        torch.cuda._sleep(400_000)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        pf.deliver(w, pf.ResamplerConfig("systematic"), pf.RngStream(r), index_dtype=torch.int32, out=c)
        e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"deliver 2^24 {dt.__name__}: median {np.median(ts):.1f} us  min {np.min(ts):.1f} us", flush=True)
sys.exit(1 if fails else 0)
