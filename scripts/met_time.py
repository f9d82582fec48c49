"""CUDA-event timing of the fused Metropolis delivery (B=32, N=2^20 log-normal
sigma=1; L2 flushed).  Usage: [PFR_MET_TABLE=0] [PFR_MET_VARIANT=1] python scripts/met_time.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402

torch.cuda.set_device(0)
pf.config.check = False
n = int(os.environ.get("N", 1 << 20))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
g = np.random.default_rng(0)
lw = g.normal(0, 1, n)
for dt in (np.float32, np.float64):
    w = torch.from_numpy(np.exp(lw - lw.max()).astype(dt)).cuda()
    c = torch.empty(n, dtype=torch.int32, device="cuda")
    ts = []
    for r in range(15):
        flush.zero_()
        torch.cuda._sleep(400_000)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        pf.deliver(w, pf.ResamplerConfig("metropolis", b=32), pf.RngStream(r), index_dtype=torch.int32, out=c)
        e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"metropolis delivery {np.dtype(dt).name} 2^{int(np.log2(n))}: median {np.median(ts):.1f} us "
          f"min {np.min(ts):.1f}", flush=True)
