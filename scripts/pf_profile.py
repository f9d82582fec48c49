"""A short batched-filter run for ncu: 512 filters x 2^16 particles, T=12."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402
from oracle.pf_oracle import simulate_observations  # noqa: E402
from paper_1301_4019_b200.pf import LinearGaussianModel  # noqa: E402

m = LinearGaussianModel(coeff=0.9)
filters = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ys = np.stack([simulate_observations(m, 12, k) for k in range(filters)])
pf.pf_run(m, ys, 1 << 16, seed=1)
print("done")
