import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf
from paper_1301_4019_b200 import _lib as L
pf.config.check = False
for logn in (16, 20, 24):
    n = 1 << logn
    g = np.random.default_rng(1); lw = g.normal(0, 1, n)
    for dt in (np.float32, np.float64):
        w = torch.from_numpy(np.exp(lw - lw.max()).astype(dt)).cuda()
        rs = pf.RngStream(3)
        st = L.status_word(); st.zero_()
        c, steps = pf.deliver(w, pf.ResamplerConfig("systematic"), rs, index_dtype=torch.int32, return_max_steps=True)
        torch.cuda.synchronize()
        flags = L._ws[0][:8].view(torch.int32).cpu().numpy()
        bits = L.read_status(st)
        O_old = pf.systematic_cumulative_offspring(w, rs, index_dtype=torch.int32)
        c_old, s_old = pf.permute_cumulative(O_old, return_max_steps=True, index_dtype=torch.int32)
        print(f"2^{logn} {dt.__name__}: dv state={flags} status={bits:#x} steps={steps}/{s_old} "
              f"equal={torch.equal(c, c_old)}", flush=True)
