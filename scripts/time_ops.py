"""CUDA-event timing of single operations (L2 flushed before each rep).
usage: python scripts/time_ops.py <op> [log2n] [dtype]   op: rejection | metropolis | systematic | multinomial
With no arguments: a sweep of the profiling knobs (PFR_REJ_BATCH) in subprocesses."""
import os
import subprocess
import sys

if len(sys.argv) == 1:
    for b in ("2", "4", "8"):
        for dt in ("f32", "f64"):
            env = dict(os.environ, PFR_REJ_BATCH=b)
            r = subprocess.run([sys.executable, __file__, "rejection", "20", dt], env=env, capture_output=True, text=True)
            print(f"rejection batch={b} {dt}: {r.stdout.strip()} {r.stderr.strip()[-300:]}")
    sys.exit(0)
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402

op = sys.argv[1]
n = 1 << int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
dt = np.float64 if (len(sys.argv) > 3 and sys.argv[3] == "f64") else np.float32
pf.config.check = False
g = np.random.default_rng(1)
lw = g.normal(0, float(os.environ.get("SIGMA", "1")), n)
w = torch.from_numpy(np.exp(lw - lw.max()).astype(dt)).cuda()
sup = float(w.max())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
c = torch.empty(n, dtype=torch.int32, device="cuda")
ts = []
for r in range(13):
    flush.zero_()
    torch.cuda._sleep(400_000)  # ~200 us: the host enqueues the work while the GPU spins
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    if op == "rejection":
        pf.rejection_ancestors(w, sup, pf.RngStream(r), index_dtype=torch.int32)
    elif op == "metropolis":
        pf.metropolis_ancestors(w, 32, pf.RngStream(r), index_dtype=torch.int32)
    elif op == "multinomial":
        pf.multinomial_ancestors(w, pf.RngStream(r), index_dtype=torch.int32)
    elif op == "systematic":
        pf.deliver(w, pf.ResamplerConfig("systematic"), pf.RngStream(r), index_dtype=torch.int32, out=c)
    e1.record()
    torch.cuda.synchronize()
    if r >= 3:
        ts.append(e0.elapsed_time(e1) * 1e3)
print(f"median {np.median(ts):.1f} us  min {np.min(ts):.1f} us")
