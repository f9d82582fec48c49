"""CUDA-event timing of the own-stream multinomial delivery (N=2^20 log-normal
sigma=1; L2 flushed)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402

torch.cuda.set_device(0)
pf.config.check = False
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for lg in [int(x) for x in os.environ.get("LOGN", "20 24").split()]:
    n = 1 << lg
    lw = np.random.default_rng(0).normal(0, 1, n)
    for dt in (np.float32, np.float64):
        w = torch.from_numpy(np.exp(lw - lw.max()).astype(dt)).cuda()
        c = torch.empty(n, dtype=torch.int32, device="cuda")
        for what in ("ancestors", "delivery"):
            ts = []
            for r in range(12):
                flush.zero_()
                torch.cuda._sleep(400_000)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                if what == "delivery":
                    pf.deliver(w, pf.ResamplerConfig("multinomial"), pf.RngStream(r), index_dtype=torch.int32, out=c)
                else:
                    pf.multinomial_ancestors(w, pf.RngStream(r), index_dtype=torch.int32)
                e1.record()
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(e0.elapsed_time(e1) * 1e3)
            print(f"multinomial {what} {np.dtype(dt).name} 2^{lg}: median {np.median(ts):.1f} us", flush=True)
