"""Rejection paths under compute-sanitizer: the certain-reject table (g = 1,
2), the plain kernel (tiny N), capped, the tail helpers."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402

for n in (100, 8192, 70001, (1 << 20) + 7):
    for dt in (np.float32, np.float64):
        g = np.random.default_rng(n)
        w = np.exp(g.normal(0, 1, n)).astype(dt)
        a, t = pf.rejection_ancestors(w, float(w.max()), pf.RngStream(1), return_trips=True)
        a2, ow = pf.rejection_ancestors_capped(w, float(np.median(w)), pf.RngStream(2))
        assert int(a.min()) >= 0 and int(a.max()) < n and int(a2.max()) < n
print("sanitize_rejection ok")
