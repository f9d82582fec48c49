"""Host-side (enqueue) cost of the public API calls, N=2^20: wall time per
call with the GPU kept busy (no syncs inside the loop), plus a cProfile of
the slowest call."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402

pf.config.check = False
n = 1 << 20
g = np.random.default_rng(0)
w = torch.from_numpy(np.exp(g.normal(0, 1, n))).cuda()
out = torch.empty(n, dtype=torch.int32, device="cuda")
sup = float(w.max())
calls = {
    "systematic": lambda r: pf.deliver(w, pf.ResamplerConfig("systematic"), pf.RngStream(r), index_dtype=torch.int32,
                                       out=out),
    "multinomial": lambda r: pf.multinomial_ancestors(w, pf.RngStream(r), index_dtype=torch.int32),
    "metropolis": lambda r: pf.metropolis_ancestors(w, 32, pf.RngStream(r), index_dtype=torch.int32),
    "rejection": lambda r: pf.rejection_ancestors(w, sup, pf.RngStream(r), index_dtype=torch.int32),
    "permute": lambda r: pf.permute_parallel(out, index_dtype=torch.int32),
    "rngstream": lambda r: pf.RngStream(r, (1, 2, 3)),
}
for name, fn in calls.items():
    for r in range(3):
        fn(r)
    torch.cuda.synchronize()
    torch.cuda._sleep(2_000_000_000 // 1000 * 50)  # keep the GPU busy so enqueue never blocks
    t0 = time.perf_counter()
    for r in range(20):
        fn(r)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:12s} {1e6 * (t1 - t0) / 20:8.1f} us/call (host)", flush=True)
torch.cuda._sleep(100_000_000)
pr = cProfile.Profile()
pr.enable()
for r in range(20):
    calls["metropolis"](r)
    calls["permute"](r)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
