"""Worker for tests/test_sharded.py::test_gpu_sharded_real_processes: the
sharded deliveries over real processes (gloo payloads in host memory, the
kernels of every rank on one GPU), compared on rank 0 with the single-GPU
delivery.  python -m torch.distributed.run --nproc-per-node P tests/shard_gloo_worker.py [log2n]"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402
from paper_1301_4019_b200 import sharded  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n = 1 << log2n
g = np.random.default_rng(5)
w_full = np.exp(g.normal(0, 1, n)).astype(np.float32)
cuts = [n * r // world for r in range(world + 1)]  # uneven shards when world does not divide n
w = torch.from_numpy(w_full[cuts[rank]:cuts[rank + 1]].copy()).cuda()
comm = sharded.DistComm()
ops = sharded.CudaShardOps()
sup_v = float(np.quantile(w_full, 0.95))
for alg in ("systematic", "stratified", "metropolis", "rejection", "rejection-capped", "multinomial"):
    cfg = pf.ResamplerConfig(alg, b=8 if alg == "metropolis" else None,
                             sup_v=sup_v if alg == "rejection-capped" else None)
    c = sharded.deliver_sharded(w, cfg, pf.RngStream(3), comm=comm, ops=ops)
    torch.cuda.synchronize()
    parts = [None] * world
    dist.all_gather_object(parts, c.cpu().numpy())
    if rank == 0:
        full = np.concatenate(parts)
        single = pf.deliver(torch.from_numpy(w_full).cuda(), cfg, pf.RngStream(3)).cpu().numpy()
        print(alg, "identical" if np.array_equal(full, single) else "DIFFERENT", flush=True)
dist.barrier()
dist.destroy_process_group()
