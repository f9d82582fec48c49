"""Every public GPU path once at small sizes (for compute-sanitizer runs):
python scripts/sanitize_paths.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402
from oracle.pf_oracle import simulate_observations  # noqa: E402
from paper_1301_4019_b200.pf import LinearGaussianModel  # noqa: E402

g = np.random.default_rng(0)
for n in (37, 5000, 70001):
    for dt in (np.float32, np.float64):
        w = torch.from_numpy(np.exp(g.normal(0, 1, n)).astype(dt)).cuda()
        for alg in ("multinomial", "stratified", "systematic"):
            pf.deliver(w, pf.ResamplerConfig(alg), pf.RngStream(1))
            pf.resample_ancestors(w, pf.ResamplerConfig(alg), pf.RngStream(2), rng_mode="numpy")
        pf.deliver(torch.log(w), pf.ResamplerConfig("systematic"), pf.RngStream(1), log_weights=True)
        pf.deliver(w, pf.ResamplerConfig("metropolis", b=8), pf.RngStream(3))
        pf.deliver(w, pf.ResamplerConfig("rejection"), pf.RngStream(4))
        pf.rejection_ancestors_capped(w, float(w.median()), pf.RngStream(5))
        a = pf.multinomial_ancestors(w, pf.RngStream(6))
        o = pf.ancestors_to_offspring(a)
        O = pf.offspring_to_cumulative(o)
        pf.cumulative_offspring_to_ancestors(O)
        pf.cumulative_to_offspring(O)
        pf.prepermute(a)
        pf.permute_parallel(a, return_max_steps=True)
        pf.permute_cumulative(O)
        pf.satisfies_inplace_predicate(pf.permute_parallel(a))
        pf.inclusive_prefix_sum(w)
        pf.exclusive_prefix_sum(w)
        pf.stable_sum(w)
        pf.ess(w)
        pf.logweights_to_weights(torch.log(w))
pf.deliver_batched(torch.rand(6, 3000, dtype=torch.float64).cuda(), pf.RngStream(7))
m = LinearGaussianModel(coeff=0.9)
ys = np.stack([simulate_observations(m, 6, k) for k in range(4)])
for n in (4096, 1000, 4096 + 32):
    pf.pf_run(m, ys, n, seed=1)
torch.cuda.synchronize()
print("all paths ran")
