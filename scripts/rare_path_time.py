"""Wall time of deliveries that need the rare path (an N-2 loser chain:
w = (2, 1, ..., 1, 0)) on the 16-CTA cooperative grid, against a regular
delivery of the same size.  Usage: python scripts/rare_path_time.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402

torch.cuda.set_device(0)
for lg in (20, 22, 24):
    n = 1 << lg
    w = torch.ones(n, dtype=torch.float32, device="cuda")
    w[0], w[-1] = 2.0, 0.0
    wr = torch.from_numpy(np.exp(np.random.default_rng(0).normal(0, 1, n)).astype(np.float32)).cuda()
    for name, x in (("regular", wr), ("rare path", w)):
        pf.deliver(x, pf.ResamplerConfig("systematic"), pf.RngStream(0))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        c = pf.deliver(x, pf.ResamplerConfig("systematic"), pf.RngStream(1))
        torch.cuda.synchronize()
        print(f"2^{lg} {name}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
