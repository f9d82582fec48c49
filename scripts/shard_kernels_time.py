"""Device time of the sharded v3 per-rank kernels alone (pfr_shard_local_end,
pfr_shard_produce, pfr_shard_resolve_fast; no collectives): one shard of
2^k float32 weights as the middle rank of a larger vector, L2 flushed.
The basis of DESIGN 4's model for config 4 on 8 GPUs."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402
from paper_1301_4019_b200 import sharded  # noqa: E402

torch.cuda.set_device(0)
pf.config.check = False
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 25
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n_loc = 1 << lg
n = n_loc * world
rank = world // 2
base = rank * n_loc
w = torch.exp(torch.randn(n_loc, device="cuda")).float()
ops = sharded.CudaShardOps()
halo = sharded.halo_width(n)
slot_lo = ((base - halo) // 4) * 4
slot_hi = base + n_loc + halo
ext = torch.empty(slot_hi - slot_lo, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
end0 = ops.local_end(w)
# a plausible prefix / total for a middle shard: the other shards weigh the same
pt = torch.tensor([float(end0) * rank, float(end0) * world], dtype=torch.float64, device="cuda")
ts = []
for r in range(12):
    flush.zero_()
    torch.cuda._sleep(300_000)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.local_end(w)
    ops.shard_produce(w, base, n, pt, False, False, False, 0.37, None, pf.RngStream(1), "philox", ext, slot_lo, slot_hi)
    c, st = ops.shard_resolve_fast(ext, slot_lo, slot_hi, base, n_loc, torch.float32)
    e1.record()
    torch.cuda.synchronize()
    if r >= 2:
        ts.append(e0.elapsed_time(e1) * 1e3)
print(f"sharded v3 per-rank kernels, shard 2^{lg} f32 of 2^{int(math.log2(n))} ({world} ranks): "
      f"median {np.median(ts):.1f} us (halo {halo} slots)")
