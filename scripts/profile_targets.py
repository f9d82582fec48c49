"""Launch the north-star paths at N=2^24 f32 (DT=f64: float64 weights) for ncu (a few reps each)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 24
pf.config.check = False
g = np.random.default_rng(1)
lw = g.normal(0, 1, n)
w = torch.from_numpy(np.exp(lw - lw.max()).astype(np.float64 if os.environ.get("DT") == "f64" else np.float32)).cuda()
c = torch.empty(n, dtype=torch.int32, device="cuda")
for r in range(reps):
    if which in ("all", "systematic"):
        pf.deliver(w, pf.ResamplerConfig("systematic"), pf.RngStream(r), index_dtype=torch.int32, out=c)
    if which in ("all", "metropolis"):
        a = pf.metropolis_ancestors(w, 32, pf.RngStream(r), index_dtype=torch.int32)
        pf.permute_parallel(a, index_dtype=torch.int32)
    if which in ("all", "rejection"):
        a = pf.rejection_ancestors(w, float(w.max()), pf.RngStream(r), index_dtype=torch.int32)
    if which in ("all", "multinomial"):
        pf.deliver(w, pf.ResamplerConfig("multinomial"), pf.RngStream(r), index_dtype=torch.int32, out=c)
    if which in ("all", "metropolis-delivery"):
        pf.deliver(w, pf.ResamplerConfig("metropolis", b=32), pf.RngStream(r), index_dtype=torch.int32, out=c)
    if which in ("all", "stratified"):
        pf.deliver(w, pf.ResamplerConfig("stratified"), pf.RngStream(r), index_dtype=torch.int32, out=c)
torch.cuda.synchronize()
print("done")
