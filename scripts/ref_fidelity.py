"""Reference-arm fidelity (dev container only: imports the read-only reference).

Times every delivery of the bench step (5 resamplers x f32/f64 at N=2^20,
log-normal sigma=1, sup_w = max w, Metropolis B=32) through the REAL
reference (resample_ancestors + permute_parallel, bench.py:155-161) and
through the oracle port (oracle/pfr_oracle.py deliver), best of 3 each, one
process, and prints the port/reference time ratio per delivery.  The bench's
reference arm times the port; this shows the port is a faithful stand-in.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from oracle import pfr_oracle as orc  # noqa: E402

import pfresample.ancestry as ranc  # noqa: E402
from pfresample.resamplers import ResamplerConfig, resample_ancestors  # noqa: E402
from pfresample.rng import RngStream  # noqa: E402

N = int(os.environ.get("N", 1 << 20))
REPS = int(os.environ.get("REPS", 3))


def best(fn):
    ts = []
    for _ in range(REPS):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def main():
    g = np.random.default_rng(0)
    lw = g.normal(0.0, 1.0, N)
    rows = []
    for dt in (np.float32, np.float64):
        w = np.exp(lw - lw.max()).astype(dt)
        for alg in ("multinomial", "stratified", "systematic", "metropolis", "rejection"):
            kw = {"b": 32} if alg == "metropolis" else ({"sup_w": float(w.max())} if alg == "rejection" else {})
            cfg = ResamplerConfig(algorithm=alg, **kw)

            def ref():
                out = resample_ancestors(w, cfg, RngStream(7, (1,)))
                ranc.permute_parallel(out.ancestors)

            def port():
                orc.deliver(w, alg, 7, (1,), **kw)

            tr, tp = best(ref), best(port)
            rows.append((alg, np.dtype(dt).name, tr, tp))
            print(f"{alg:12s} {np.dtype(dt).name:8s} reference {tr:7.3f} s  port {tp:7.3f} s  port/ref {tp / tr:5.2f}",
                  flush=True)
    tr = sum(r[2] for r in rows)
    tp = sum(r[3] for r in rows)
    print(f"step total: reference {tr:.2f} s, port {tp:.2f} s, port/ref {tp / tr:.3f}")


if __name__ == "__main__":
    main()
