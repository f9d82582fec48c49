"""CUDA-event timing of the own-stream rejection kernel (N=2^20 log-normal
sigma=1, sup_w = max w; L2 flushed), plus mean trips per slot.
Usage: [PFR_REJ_PACK=0] [PFR_REJ_BATCH=b] python scripts/rej_time.py"""
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
    sup = float(w.max())
    ts = []
    for r in range(15):
        flush.zero_()
        torch.cuda._sleep(400_000)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        pf.rejection_ancestors(w, sup, pf.RngStream(r), index_dtype=torch.int32)
        e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"rejection {np.dtype(dt).name} 2^{int(np.log2(n))}: median {np.median(ts):.1f} us min {np.min(ts):.1f}",
          flush=True)
