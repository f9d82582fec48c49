"""Timing of the weight-sharded systematic delivery (protocol v2) with real
processes on ONE GPU (gloo): torchrun --nproc-per-node G scripts/shard_time.py [log2N].
Every rank's kernels share the one B200 and gloo moves the collectives through
host memory, so this measures the protocol's overheads, not NVLink scaling."""
import os
import statistics
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402
from paper_1301_4019_b200 import sharded  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
n = 1 << lg
n_loc = n // world
g = torch.Generator(device="cuda")
g.manual_seed(77 + rank)
w = torch.exp(torch.randn(n_loc, device="cuda", generator=g) * 1.0).float()
comm = sharded.DistComm()
ops = sharded.CudaShardOps()
for alg in ("systematic", "metropolis", "multinomial"):
    cfg = pf.ResamplerConfig(alg, b=32 if alg == "metropolis" else None)
    ts = []
    for r in range(4):
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        sharded.deliver_sharded(w, cfg, pf.RngStream(r), comm=comm, ops=ops)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    t = torch.tensor([statistics.median(ts)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"{alg} 2^{lg} f32 over {world} ranks (gloo, one GPU): {t.item():.2f} ms  "
              f"protocol counts {sharded.protocol_counts}", flush=True)
dist.destroy_process_group()
