"""CUDA-event timing of the fused delivery with only the first k kernels
(PFR_DV_STAGES) at N=2^24 f32; L2 flushed before each rep."""
import os, subprocess, sys, json
if len(sys.argv) == 1:
    for k in (1, 2, 3, 4):
        env = dict(os.environ, PFR_DV_STAGES=str(k))
        out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
        print(f"stages<={k}: {out.stdout.strip()} {out.stderr.strip()[-300:]}")
    sys.exit(0)
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf
pf.config.check = False
n = int(os.environ.get("N", 1 << 24))
dt = np.float64 if os.environ.get("DT") == "f64" else np.float32
g = np.random.default_rng(int(os.environ.get("SEED", 1))); lw = g.normal(0, 1, n)
w = torch.from_numpy(np.exp(lw - lw.max()).astype(dt)).cuda()
c = torch.empty(n, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush2 = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
ts = []
for r in range(15):
    flush.zero_()
    if os.environ.get("FLUSH") == "clean":  # evict the dirty flush lines too (read pass)
        flush2.sum()
    torch.cuda._sleep(400_000)  # ~200 us: the host enqueues the work while the GPU spins
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); pf.deliver(w, pf.ResamplerConfig("systematic"), pf.RngStream(r), index_dtype=torch.int32, out=c); e1.record()
    torch.cuda.synchronize()
    if r >= 3: ts.append(e0.elapsed_time(e1) * 1e3)
print(f"median {np.median(ts):.1f} us  min {np.min(ts):.1f} us")
