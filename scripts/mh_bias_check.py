"""Metropolis own-stream Monte Carlo at N=2^22, sigma=0.5 (the C3 sweep's
weights): mean offspring of the 256 heaviest particles over R replicates,
saved for an offline comparison with the exact 1^T P^B oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402

pf.config.check = False
n, sigma, R = 1 << 22, 0.5, int(sys.argv[1]) if len(sys.argv) > 1 else 64
g = np.random.default_rng(int(7000 + 100 * sigma))
lw = g.normal(0.0, sigma, n)
w = torch.from_numpy(np.exp(lw - lw.max()).astype(np.float32)).cuda()
K = int(sys.argv[3]) if len(sys.argv) > 3 else 256
top = torch.argsort(w, descending=True)[:K]
res = {}
steps = tuple(int(b) for b in sys.argv[2].split(",")) if len(sys.argv) > 2 else (16, 32, 64)
for B in steps:
    acc = torch.zeros(K, dtype=torch.float64, device="cuda")
    acc2 = torch.zeros(K, dtype=torch.float64, device="cuda")
    for r in range(R):
        a = pf.metropolis_ancestors(w, B, pf.RngStream(5000 + r, (5, B)), index_dtype=torch.int32)
        o = pf.ancestors_to_offspring(a, index_dtype=torch.int32)[top].double()
        acc += o
        acc2 += o * o
    res[B] = (acc / R).cpu().numpy(), (acc2 / R).cpu().numpy()
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/mh_bias_check.npz", top=top.cpu().numpy(),
         **{f"mean_{B}": m for B, (m, _) in res.items()}, **{f"sq_{B}": s for B, (_, s) in res.items()})
print("saved", {B: float(m[:8].mean()) for B, (m, _) in res.items()})
