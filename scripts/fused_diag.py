"""CUDA-event timings of the systematic delivery at several N (L2 flushed
before each rep).  Usage: [PFR_DV_PIPELINE=legacy] [DT=f64] [LOGN="20 22 24"]
python scripts/fused_diag.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402

torch.cuda.set_device(0)
pf.config.check = False
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for lg in [int(x) for x in os.environ.get("LOGN", "20 22 24").split()]:
    n = 1 << lg
    dt = np.float64 if os.environ.get("DT") == "f64" else np.float32
    w = torch.from_numpy(np.exp(np.random.default_rng(1).normal(0, 1, n)).astype(dt)).cuda()
    c = torch.empty(n, dtype=torch.int32, device="cuda")
    ts = []
    for r in range(12):
        flush.zero_()
        torch.cuda._sleep(400_000)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        pf.deliver(w, pf.ResamplerConfig("systematic"), pf.RngStream(r), index_dtype=torch.int32, out=c)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"2^{lg} {dt.__name__}: median {np.median(ts):.1f} us min {np.min(ts):.1f}", flush=True)
