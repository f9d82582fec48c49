"""Mode knobs and remaining entry points once each (for compute-sanitizer):
the batched filter's forced in-place paths, replay modes, serial variants,
slot-range rejection, the gather probe."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402
from paper_1301_4019_b200 import _lib as L  # noqa: E402
from oracle.pf_oracle import simulate_observations  # noqa: E402
from paper_1301_4019_b200.pf import LinearGaussianModel  # noqa: E402
from paper_1301_4019_b200.sharded import CudaShardOps  # noqa: E402

m = LinearGaussianModel(coeff=0.8, obs_std=0.05)
ys = np.stack([simulate_observations(m, 5, k) for k in range(3)])
for path in ("0", "1", "2", "3"):
    os.environ["PFR_PF_PATH"] = path
    pf.pf_run(m, ys, 8192, ess_threshold=1.0, seed=3)
os.environ.pop("PFR_PF_PATH")
g = np.random.default_rng(2)
for n in (1 << 12, 3000):
    w = np.exp(g.normal(0, 1, n))
    pf.deliver(w, pf.ResamplerConfig("stratified"), pf.RngStream(1), rng_mode="numpy")
    pf.multinomial_ancestors(w, pf.RngStream(2), rng_mode="numpy")
    pf.multinomial_ancestors_serial(w, pf.RngStream(2), rng_mode="numpy")
    pf.metropolis_ancestors(w, 5, pf.RngStream(3), rng_mode="numpy") if n == 1 << 12 else None
    pf.permute_serial(g.integers(0, n, n))
    u = g.random((4, n))
    j = g.integers(0, n, (4, n))
    pf.metropolis_ancestors(w, 4, None, u_draws=u, j_draws=j)
ops = CudaShardOps()
w = torch.from_numpy(np.exp(g.normal(0, 1, 5000))).cuda()
ops.rejection_range(w, pf.ResamplerConfig("rejection"), pf.RngStream(4), None, 1000, 2500)
buf = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
sink = torch.zeros(1, dtype=torch.int64, device="cuda")
L.call("pfr_probe_gather", buf.data_ptr(), 1 << 16, 4, 1 << 22, sink.data_ptr(), L.stream_handle())
torch.cuda.synchronize()
print("all mode paths ran")
