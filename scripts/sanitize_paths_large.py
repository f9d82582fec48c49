"""The rare and multi-group paths once each (for compute-sanitizer runs):
multi-group tile hierarchy (N = 2^19), near-uniform weights (long K3 chains
-> the rare path's pointer jumping), an adversarial ancestry (the general
permute's fallback), the weight-sharded delivery over virtual ranks."""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402
from paper_1301_4019_b200.sharded import CudaShardOps, ThreadComm, deliver_sharded  # noqa: E402

g = np.random.default_rng(0)
n = 1 << 19
for dt in (np.float32, np.float64):
    w = torch.from_numpy(np.exp(g.normal(0, 1, n)).astype(dt)).cuda()
    pf.deliver(w, pf.ResamplerConfig("systematic"), pf.RngStream(1))
    pf.deliver(w, pf.ResamplerConfig("stratified"), pf.RngStream(1), rng_mode="numpy")
    pf.inclusive_prefix_sum(w)
wu = torch.from_numpy(np.exp(g.normal(0, 0.01, n))).cuda()  # chains of thousands of steps
pf.deliver(wu, pf.ResamplerConfig("systematic"), pf.RngStream(3), return_max_steps=True)
m = 20000
o = np.ones(m, dtype=np.int64)
o[0], o[-1] = 2, 0  # one chain of m-2 steps
a = torch.from_numpy(np.repeat(np.arange(m), o)).cuda()
pf.permute_parallel(a, return_max_steps=True)
pf.permute_cumulative(torch.from_numpy(np.cumsum(o)).cuda(), return_max_steps=True)
# weight-sharded delivery, 3 virtual ranks (one thread each)
w = np.exp(g.normal(0, 1, 300001)).astype(np.float32)
cuts = [0, 100000, 100001, 300001]
comms = ThreadComm.group(3)
outs = [None] * 3


def body(r):
    shard = torch.from_numpy(w[cuts[r]: cuts[r + 1]].copy())
    outs[r] = deliver_sharded(shard, pf.ResamplerConfig("systematic"), pf.RngStream(5), comm=comms[r],
                              ops=CudaShardOps())


def run3(fn):
    ts = [threading.Thread(target=fn, args=(r,)) for r in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


run3(body)
# the v2 protocol's general fallback (zero halo), and the slot-partitioned
# multinomial / rejection with the partitioned permute
os.environ["PFR_SHARD_HALO"] = "0"
run3(body)
del os.environ["PFR_SHARD_HALO"]


def body2(r):
    shard = torch.from_numpy(w[cuts[r]: cuts[r + 1]].copy())
    for alg in ("multinomial", "rejection"):
        outs[r] = deliver_sharded(shard, pf.ResamplerConfig(alg), pf.RngStream(6), comm=comms[r], ops=CudaShardOps(),
                                  rng_mode="philox")


run3(body2)
torch.cuda.synchronize()
print("all rare paths ran", [int(x.numel()) for x in outs])
