"""Device time of pf_run for F filters x 2^16 particles x T steps (CUDA events)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402
from oracle.pf_oracle import simulate_observations  # noqa: E402
from paper_1301_4019_b200.pf import LinearGaussianModel  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 512
T = int(sys.argv[2]) if len(sys.argv) > 2 else 100
m = LinearGaussianModel(coeff=0.9)
ys = np.stack([simulate_observations(m, T, k) for k in range(F)])
pf.pf_run(m, ys[:, :3], 1 << 16, seed=1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
res = pf.pf_run(m, ys, 1 << 16, seed=7)
e1.record()
torch.cuda.synchronize()
print(f"{F} filters x 2^16 x T={T}: {e0.elapsed_time(e1):.1f} ms, resampled {res.resampled.mean():.2f}")
