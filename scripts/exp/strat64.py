import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1301_4019_b200 as pf
w = torch.from_numpy(np.random.default_rng(0).random(64)).cuda()
c = pf.deliver(w, pf.ResamplerConfig("stratified"), pf.RngStream(1), index_dtype=torch.int32)
print(c.cpu().numpy()[:10])
