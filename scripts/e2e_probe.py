"""e2e pipeline probe: the bench's 10-delivery mix (N=2^20) back to back with
(a) weights already on the device, (b) pinned-host uploads/downloads on one
copy stream, (c) on two copy streams.  Device time per step (CUDA events)."""
import os
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
jobs = [(alg, dt) for alg in ("multinomial", "stratified", "systematic", "metropolis", "rejection") for dt in ("f32", "f64")]
dw = [host[dt].cuda() for (_, dt) in jobs]
dc = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in jobs]
hc = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in jobs]
stream = torch.cuda.current_stream()


def delivery(alg, dt, w, r, out):
    if alg in ("systematic", "stratified"):
        return pf.deliver(w, pf.ResamplerConfig(alg), pf.RngStream(r), index_dtype=torch.int32, out=out)
    if alg == "multinomial":
        a = pf.multinomial_ancestors(w, pf.RngStream(r), index_dtype=torch.int32)
    elif alg == "metropolis":
        a = pf.metropolis_ancestors(w, 32, pf.RngStream(r), index_dtype=torch.int32)
    else:
        a = pf.rejection_ancestors(w, sup[dt], pf.RngStream(r), index_dtype=torch.int32)
    return pf.permute_parallel(a, index_dtype=torch.int32)


order_cost = {"rejection": 5, "metropolis": 4, "multinomial": 3, "stratified": 2, "systematic": 1}
jobs_sorted = sorted(jobs, key=lambda j: (-order_cost[j[0]], j[1] != "f64"))
import time as _time


for variant in ("uploads", "downloads", "both", "device", "one", "one-sorted", "two-sorted"):
    if variant.endswith("sorted"):
        jobs[:] = jobs_sorted
    if variant == "both":
        sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
        ts = []
        for it in range(5):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e2 = torch.cuda.Event(enable_timing=True)
            e0.record(sa)
            sb.wait_event(e0)
            with torch.cuda.stream(sa):
                for k, (alg, dt) in enumerate(jobs):
                    dw[k].copy_(host[dt], non_blocking=True)
            with torch.cuda.stream(sb):
                for k, (alg, dt) in enumerate(jobs):
                    hc[k].copy_(dc[k], non_blocking=True)
            e1.record(sa)
            e2.record(sb)
            torch.cuda.synchronize()
            ts.append(max(e0.elapsed_time(e1), e0.elapsed_time(e2)))
        print(variant, " ".join(f"{t:.3f}" for t in ts[1:]), "ms", flush=True)
        continue
    if variant in ("uploads", "downloads"):
        st = torch.cuda.Stream()
        ts = []
        for it in range(5):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            with torch.cuda.stream(st):
                for k, (alg, dt) in enumerate(jobs):
                    if variant == "uploads":
                        dw[k].copy_(host[dt], non_blocking=True)
                    else:
                        hc[k].copy_(dc[k], non_blocking=True)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(variant, " ".join(f"{t:.3f}" for t in ts[1:]), "ms", flush=True)
        continue
    up = torch.cuda.Stream()
    down = up if variant.startswith("one") else torch.cuda.Stream()
    ts = []
    for it in range(6):
        torch.cuda.synchronize()
        up.wait_stream(stream)
        down.wait_stream(stream)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if variant == "device":
            e0.record(stream)
            for k, (alg, dt) in enumerate(jobs):
                delivery(alg, dt, dw[k], it * 100 + k, dc[k])
            e1.record(stream)
        else:
            e0.record(up)
            evs = []
            for k, (alg, dt) in enumerate(jobs):
                with torch.cuda.stream(up):
                    dw[k].copy_(host[dt], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(up)
                evs.append(ev)
            for k, (alg, dt) in enumerate(jobs):
                stream.wait_event(evs[k])
                c = delivery(alg, dt, dw[k], it * 100 + k, dc[k])
                done = torch.cuda.Event()
                done.record(stream)
                c.record_stream(down)
                with torch.cuda.stream(down):
                    down.wait_event(done)
                    hc[k].copy_(c, non_blocking=True)
            e1.record(down)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(variant, " ".join(f"{t:.3f}" for t in ts[1:]), "ms", flush=True)
