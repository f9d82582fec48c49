"""A/B of the general permute at N=2^20 / 2^24 (Metropolis B=32 ancestry):
pfr_permute (claims + forward loser walks) vs pfr_permute_range over the whole
index range (claims + backward walks from the holes).  CUDA events, L2 flushed."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402
from paper_1301_4019_b200.sharded import CudaShardOps  # noqa: E402

torch.cuda.set_device(0)
pf.config.check = False
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ops = CudaShardOps()
for lg in (20, 24):
    n = 1 << lg
    w = torch.exp(torch.randn(n, device="cuda")).float()
    a = pf.metropolis_ancestors(w, 32, pf.RngStream(1), index_dtype=torch.int32)
    want = pf.permute_parallel(a, index_dtype=torch.int32)
    c2, _, fl = ops.permute_range(a, 0, n)
    assert torch.equal(c2, want), "range permute differs"
    for name, fn in (("permute (claims + forward walks)", lambda: pf.permute_parallel(a, index_dtype=torch.int32)),
                     ("permute_range (claims + backward walks)", lambda: ops.permute_range(a, 0, n))):
        ts = []
        for r in range(12):
            flush.zero_()
            torch.cuda._sleep(200_000)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1) * 1e3)
        print(f"2^{lg} {name}: median {np.median(ts):.1f} us", flush=True)
