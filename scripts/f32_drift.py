"""The paper's fp32 prefix-sum instability on the GPU: systematic O from
float32 weights with float32 accumulation (accum='native', the reference's
np.cumsum behaviour) vs float64 accumulation (the default), against the
float64 exact positions: max |dO| and max per-parent |o - N w/W|."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402

for log2n in (16, 20, 22, 24):
    n = 1 << log2n
    g = np.random.default_rng(log2n)
    w = np.exp(g.normal(0, 1, n)).astype(np.float32)
    wt = torch.from_numpy(w).cuda()
    ref = np_ref = None
    out = {}
    for acc in ("native", "f64"):
        O_ = pf.systematic_cumulative_offspring(wt, pf.RngStream(1), offset=0.5, accum=acc).cpu().numpy()
        out[acc] = O_
    w64 = w.astype(np.float64)
    exact = np.minimum(n, np.floor(np.cumsum(w64) * n / w64.sum() + 0.5)).astype(np.int64)
    exact[-1] = n
    m = n * w64 / w64.sum()
    row = []
    for acc in ("native", "f64"):
        O_ = out[acc].astype(np.int64)
        o = np.diff(np.concatenate(([0], O_)))
        row.append(f"{acc}: max|dO|={int(np.abs(O_ - exact).max())} max|o-Nw|={np.abs(o - m).max():.2f}")
    print(f"N=2^{log2n}  " + "  ".join(row), flush=True)
