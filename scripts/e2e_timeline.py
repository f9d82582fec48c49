"""e2e timeline: the bench's concurrent step fed from pinned host buffers,
with an event after every upload, delivery and download (ms after start)."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf  # noqa: E402

pf.config.check = False
n = 1 << 20
g = np.random.default_rng(0)
lw = g.normal(0, 1, n)
w64 = np.exp(lw - lw.max())
host = {"f32": torch.from_numpy(w64.astype(np.float32)).pin_memory(), "f64": torch.from_numpy(w64).pin_memory()}
sup = {k: float(v.max()) for k, v in host.items()}
order = os.environ.get("ORDER", "long")
algs = ("rejection", "metropolis", "multinomial", "stratified", "systematic")
if order == "short":
    algs = algs[::-1]
jobs = [(a, d) for a in algs for d in ("f64", "f32")]
if order == "mixed":  # one long, one short, alternating
    long_, short = jobs[:4], jobs[4:][::-1]
    jobs = [x for pair in zip(short[:4], long_) for x in pair] + short[4:]
dw = [host[dt].cuda() for (_, dt) in jobs]
dc = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in jobs]
hc = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in jobs]
streams = [torch.cuda.Stream() for _ in jobs]
up_s, down_s = torch.cuda.Stream(), torch.cuda.Stream()
cur = torch.cuda.current_stream()


def delivery(alg, dt, w, r, out):
    if alg in ("systematic", "stratified", "metropolis"):
        return pf.deliver(w, pf.ResamplerConfig(alg, b=32), pf.RngStream(r), index_dtype=torch.int32, out=out)
    if alg == "multinomial":
        a = pf.multinomial_ancestors(w, pf.RngStream(r), index_dtype=torch.int32)
    else:
        a = pf.rejection_ancestors(w, sup[dt], pf.RngStream(r), index_dtype=torch.int32)
    return pf.permute_parallel(a, index_dtype=torch.int32)


def ev(s):
    e = torch.cuda.Event(enable_timing=True)
    e.record(s)
    return e


for it in range(4):
    torch.cuda.synchronize()
    torch.cuda._sleep(4_000_000)
    up_s.wait_stream(cur)
    down_s.wait_stream(cur)
    e0 = ev(up_s)
    ups, dels, downs = [], [], []
    for k, (alg, dt) in enumerate(jobs):
        with torch.cuda.stream(up_s):
            dw[k].copy_(host[dt], non_blocking=True)
            ups.append(ev(up_s))
    for k, (alg, dt) in enumerate(jobs):
        streams[k].wait_event(ups[k])
        with torch.cuda.stream(streams[k]):
            c = delivery(alg, dt, dw[k], it * 10 + k, dc[k])
            dels.append(ev(streams[k]))
        c.record_stream(down_s)
        with torch.cuda.stream(down_s):
            down_s.wait_event(dels[k])
            hc[k].copy_(c, non_blocking=True)
            downs.append(ev(down_s))
    torch.cuda.synchronize()
    if it == 3:
        print(f"{order} iter {it}: uploads done {ups[-1].elapsed_time(e0) * -1 if False else e0.elapsed_time(ups[-1]):.3f}  "
              f"deliveries done {max(e0.elapsed_time(e) for e in dels):.3f}  downloads done "
              f"{max(e0.elapsed_time(e) for e in downs):.3f} ms")
        if os.environ.get("VERBOSE"):
          print("   per job (upload end, delivery end, download end):",
              [(a[:4] + d, round(e0.elapsed_time(u), 2), round(e0.elapsed_time(dl), 2), round(e0.elapsed_time(dn), 2))
               for (a, d), u, dl, dn in zip(jobs, ups, dels, downs)])
