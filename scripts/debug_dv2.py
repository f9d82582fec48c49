import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf
from paper_1301_4019_b200 import _lib as L
pf.config.check = False
n = 1 << 16
g = np.random.default_rng(1); lw = g.normal(0, 1, n)
w = torch.from_numpy(np.exp(lw - lw.max())).cuda()
c = pf.deliver(w, pf.ResamplerConfig("systematic"), pf.RngStream(3), index_dtype=torch.int32)
torch.cuda.synchronize()
st = L._ws[0][:256].view(torch.int64).cpu().numpy()
print("state", st[:2], "dbg", st[1:24].tolist())
O = pf.systematic_cumulative_offspring(w, pf.RngStream(3), index_dtype=torch.int32).cpu().numpy()
base, tid = int(st[2]), int(st[3])
print("true O at thread:", O[base + 16*tid - 1: base + 16*tid + 16].tolist())
