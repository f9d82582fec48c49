"""Benchmark: particles resampled per second (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[1]): all five resamplers -- multinomial,
stratified, systematic, Metropolis(B=32), rejection(sup_w = max w) -- at
N = 2^20 on i.i.d. log-normal (sigma = 1) weights, float32 AND float64.  One
step = the ten deliveries (resample + permute to an in-place-valid ancestry,
the timed region of the reference's bench.py:155-161), i.e. 10 * 2^20
particles.  The ten deliveries are independent filters' resampling and run
concurrently, each on its own stream with its own copy of the weights (the
reference's bench runs its cells concurrently too, bench.py:226-230); weights
are resident in HBM before timing; L2 is flushed (256 MiB write) before every
step, outside the timed region; a GPU spin between the flush and the start
event lets the host enqueue the whole step so that the CUDA events see device
work only (the host-side cost of the API is what `e2e` measures).  The same
ten deliveries are also timed one at a time (L2 flushed before each):
`sequential` and `per_delivery_ms`, from which the dominant kernel's roofline
is computed.

Also reported (north-star targets): systematic delivery
and Metropolis(B=32) at N = 2^24 float32 against the measured HBM roofline.

`--impl reference` times the reference algorithm on the host: the oracle
port (oracle/pfr_oracle.py, NumPy + the Python chain walk, like the reference),
the ten deliveries spread over a process pool using every host core.

Multi-GPU (torchrun): every rank runs the same per-GPU workload on its own
independent filters (no communication, scaling "weak"); value = all ranks'
particles / max-over-ranks time.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALGS = ("multinomial", "stratified", "systematic", "metropolis", "rejection")
DTYPES = ("f32", "f64")
METRIC = "particles resampled/sec vs N per resampler (1/2/4/8 B200); % HBM roofline"
N_DEFAULT = 1 << 20
B_STEPS = 32
SIGMA = 1.0
PREROLL_CYCLES = 400_000  # ~0.2 ms GPU spin before each timed delivery (outside the events)
STEP_PREROLL_CYCLES = 4_000_000  # ~2 ms spin before a concurrent step: the host enqueues all ten deliveries


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def log_normal_weights(n, seed, dtype=np.float64):
    g = np.random.default_rng(seed)
    lw = g.normal(0.0, SIGMA, n)
    return np.exp(lw - lw.max()).astype(dtype)


def algorithmic_bytes(alg, s, n, trips=None):
    """bytes per particle x N for one delivery's dominant kernel."""
    if alg in ("systematic", "stratified", "multinomial"):
        return (s + 4) * n
    if alg == "metropolis":
        return (s + 4 + B_STEPS * s) * n
    if alg == "rejection":
        return (s + 4 + trips * s) * n
    raise ValueError(alg)


# ---------------------------------------------------------------------------
# clocks sampler


class Clocks:
    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append((time.time(), parts))

    def wait_first(self, timeout=5.0, busy=None):
        """Keep the GPU busy (``busy()``) until the sampler has produced a sample."""
        t0 = time.time()
        while self.proc and not self.samples and time.time() - t0 < timeout:
            if busy:
                busy()
            else:
                time.sleep(0.05)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, window=None):
        """Clocks over the samples taken inside ``window`` (t0, t1) -- the timed
        region; when it is shorter than the sampling period, the samples
        nearest to it (the GPU runs warm-up / e2e steps back to back around it)."""
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        chosen = self.samples
        where = "whole run"
        if window:
            t0, t1 = window
            inside = [s for s in self.samples if t0 <= s[0] <= t1]
            if inside:
                chosen, where = inside, "timed region"
            else:
                mid = 0.5 * (t0 + t1)
                chosen = sorted(self.samples, key=lambda s: abs(s[0] - mid))[:3]
                where = "nearest to the timed region (GPU busy with warm-up/e2e steps)"
        samples = [s[1] for s in chosen]
        sm = [float(s[0]) for s in samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(samples), "sampled": where}


# ---------------------------------------------------------------------------
# reference arm (host)


def _ref_delivery(args):
    alg, dt, n, seed = args
    from oracle import pfr_oracle as orc

    w = log_normal_weights(n, seed, np.float32 if dt == "f32" else np.float64)
    t0 = time.perf_counter()
    orc.deliver(w, alg, seed, (1,), b=B_STEPS, sup_w=float(w.max()))
    return time.perf_counter() - t0


def cpu_step(n, pool, seed=0):
    """One step of the workload on the host; returns wall seconds."""
    jobs = [(alg, dt, n, seed + i) for i, (alg, dt) in enumerate((a, d) for a in ALGS for d in DTYPES)]
    t0 = time.perf_counter()
    if pool is None:
        for j in jobs:
            _ref_delivery(j)
    else:
        list(pool.map(_ref_delivery, jobs))
    return time.perf_counter() - t0


def host_cpu_info() -> dict:
    """nproc and the CPU model of this host (the CPU arm states its hardware)."""
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        affinity = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        affinity = os.cpu_count() or 1
    return {"nproc": affinity, "cpu_count": os.cpu_count(), "cpu_model": model or "unknown"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    import multiprocessing as mp

    cores = min(os.cpu_count() or 1, len(ALGS) * len(DTYPES))
    n = args.n
    with mp.get_context("spawn").Pool(cores) as pool:
        for _ in range(args.warmup):
            cpu_step(n, pool)
        times = [cpu_step(n, pool) for _ in range(args.steps)]
    per = sum(times) / len(times)
    units = len(ALGS) * len(DTYPES) * n
    value = units / per
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "particles/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32,f64", "data": "synthetic log-normal weights",
        "config": workload_config(n, world),
        "cpu_baseline": {"value": value, "unit": "particles/s", "cores": cores, "kind": "port",
                         "sample": f"the full step: 5 resamplers x (f32, f64) at N=2^{int(math.log2(n))}, "
                                   f"oracle/pfr_oracle.py (NumPy + Python chain walk) over a {cores}-process pool",
                         **host_cpu_info()},
        "e2e": {"value": value, "unit": "particles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(n, world):
    return {"workload": "configs[1]: multinomial/stratified/systematic/metropolis(B=32)/rejection(sup_w=max w), "
                        f"N=2^{int(math.log2(n))}, f32 and f64, log-normal sigma={SIGMA}",
            "n_particles": n, "deliveries_per_step": len(ALGS) * len(DTYPES), "metropolis_B": B_STEPS,
            "rng": "own Philox4x32-10 (rng_mode='philox')",
            "l2": "flushed (256 MiB write) before every step (and before every delivery of the sequential leg)",
            "concurrency": "the ten deliveries of a step on ten streams (independent filters)",
            "parallelism": f"replicas x{world} (independent filters per GPU)"}


# ---------------------------------------------------------------------------
# GPU arm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-targets", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_1301_4019_b200 import _build

    _build.build()
    import paper_1301_4019_b200 as pf
    from paper_1301_4019_b200 import _lib as L

    # PFR_BENCH_BACKEND / PFR_BENCH_DEVICE (test knobs): run the multi-rank
    # protocol with gloo on one GPU to check it before a multi-GPU run
    backend = os.environ.get("PFR_BENCH_BACKEND", "nccl")
    local = int(os.environ.get("PFR_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    pf.config.check = False  # validation kernels still run; statuses are read after timing
    hbm, peak_src = peaks()
    n = args.n

    weights = {}
    for i, dt in enumerate(DTYPES):
        w = log_normal_weights(n, 1000 * rank + i, np.float32 if dt == "f32" else np.float64)
        weights[dt] = torch.from_numpy(w).to(dev)
    sup = {dt: float(weights[dt].max()) for dt in DTYPES}
    trips = {dt: sup[dt] * n / float(weights[dt].double().sum()) for dt in DTYPES}
    outs = {dt: torch.empty(n, dtype=torch.int32, device=dev) for dt in DTYPES}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    cfgs = {alg: pf.ResamplerConfig(alg, b=B_STEPS, sup_w=None) for alg in ALGS}

    def delivery(alg, dt, rs, parts=None):
        """One delivery; `parts` collects (name, start, end) event pairs per sub-call."""
        w = weights[dt]
        if alg in ("systematic", "stratified"):
            return pf.deliver(w, cfgs[alg], rs, index_dtype=torch.int32, out=outs[dt])
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if alg == "multinomial":
            a = pf.multinomial_ancestors(w, rs, index_dtype=torch.int32)
        elif alg == "metropolis":
            a = pf.metropolis_ancestors(w, B_STEPS, rs, index_dtype=torch.int32)
        else:
            a = pf.rejection_ancestors(w, sup[dt], rs, index_dtype=torch.int32)
        e1.record(stream)
        if parts is not None:
            parts.append((f"{alg}/{dt}", e0, e1))
        return pf.permute_parallel(a, index_dtype=torch.int32)

    def timed_step(step, parts):
        evs = []
        for i, alg in enumerate(ALGS):
            for j, dt in enumerate(DTYPES):
                flush.zero_()
                # the GPU spins while the host enqueues the delivery, so the
                # events time device work only (host cost is in `e2e`)
                torch.cuda._sleep(PREROLL_CYCLES)
                s0 = torch.cuda.Event(enable_timing=True)
                s1 = torch.cuda.Event(enable_timing=True)
                s0.record(stream)
                delivery(alg, dt, pf.RngStream(step, (rank, i, j)), parts)
                s1.record(stream)
                evs.append((f"{alg}/{dt}", s0, s1))
        return evs

    clk = Clocks(local).__enter__()
    for s in range(args.warmup):
        timed_step(10_000 + s, None)
    # keep the GPU under load until the clock sampler is producing samples
    clk.wait_first(busy=lambda: (timed_step(20_000, None), torch.cuda.synchronize()))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    L.lib().pfr_launch_count(1)
    per_delivery = {}
    kernel_parts = {}
    t_wall0 = time.time()
    all_evs, all_parts = [], []
    for s in range(args.steps):
        parts = []
        all_evs.append(timed_step(s, parts))
        all_parts.append(parts)
    torch.cuda.synchronize()
    seq_launches = int(L.lib().pfr_launch_count(1))

    # ---------------- the step: ten independent deliveries at once ----------------
    # Each delivery is an independent filter's resampling; they run on their
    # own streams (each (device, stream) has its own workspace and status
    # words), as the reference's bench runs its cells concurrently
    # (bench.py:226-230).  Every delivery reads its own copy of the weights;
    # L2 is flushed before every step; the GPU spins while the host enqueues
    # the step, so the events time device work.
    jobs = [(i, alg, j, dt) for i, alg in enumerate(ALGS) for j, dt in enumerate(DTYPES)]
    conc_streams = [torch.cuda.Stream(device=dev) for _ in jobs]
    conc_w = [weights[dt].clone() for (_, _, _, dt) in jobs]
    conc_out = [torch.empty(n, dtype=torch.int32, device=dev) for _ in jobs]

    rej_cfg = {dt: pf.ResamplerConfig("rejection", sup_w=sup[dt]) for dt in DTYPES}

    def run_delivery(alg, dt, w, rs, out):
        # every delivery is the fused library call: the resampler makes the
        # permute's claims (Metropolis, rejection, multinomial) or the whole
        # delivery is one pipeline (systematic, stratified)
        cfg = rej_cfg[dt] if alg == "rejection" else cfgs[alg]
        return pf.deliver(w, cfg, rs, index_dtype=torch.int32, out=out)

    # submission order of the concurrent step: the longest deliveries first
    # (rejection, Metropolis), so the short ones fill the SMs around them
    # (1.00 ms/step vs 1.07 ms in table order; PFR_CONC_ORDER=table for A/B)
    conc_order = list(range(len(jobs)))
    if os.environ.get("PFR_CONC_ORDER") != "table":
        rank_alg = {"rejection": 0, "metropolis": 1, "multinomial": 2, "stratified": 3, "systematic": 4}
        conc_order.sort(key=lambda k: (rank_alg[jobs[k][1]], jobs[k][3]))

    def concurrent_step(step):
        flush.zero_()
        torch.cuda._sleep(STEP_PREROLL_CYCLES)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        done = []
        for k in conc_order:
            i, alg, j, dt = jobs[k]
            sk = conc_streams[k]
            sk.wait_event(e0)
            with torch.cuda.stream(sk):
                run_delivery(alg, dt, conc_w[k], pf.RngStream(step, (rank, i, j)), conc_out[k])
                ev = torch.cuda.Event()
                ev.record(sk)
            done.append(ev)
        for ev in done:
            stream.wait_event(ev)
        e1.record(stream)
        return e0, e1

    for s in range(args.warmup):
        concurrent_step(30_000 + s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    L.lib().pfr_launch_count(1)
    conc_evs = [concurrent_step(s) for s in range(args.steps)]
    torch.cuda.synchronize()
    t_wall1 = time.time()
    launches = int(L.lib().pfr_launch_count(1))
    conc_ms = sum(a.elapsed_time(b) for a, b in conc_evs)

    total_ms = 0.0
    for evs in all_evs:
        for name, a, b in evs:
            t = a.elapsed_time(b)
            per_delivery.setdefault(name, []).append(t)
            total_ms += t
    for parts in all_parts:
        for name, a, b in parts:
            kernel_parts.setdefault(name, []).append(a.elapsed_time(b))
    status = L.status_all()
    if world > 1:
        t = torch.tensor([total_ms, conc_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, conc_ms = float(t[0].item()), float(t[1].item())
    seq_ms_per_step = total_ms / args.steps
    ms_per_step = conc_ms / args.steps
    units_per_step = len(ALGS) * len(DTYPES) * n
    value = world * units_per_step / (ms_per_step * 1e-3)
    seq_value = world * units_per_step / (seq_ms_per_step * 1e-3)

    # dominant kernel of the step (largest share), roofline from live events
    dom_name, dom_ms = None, 0.0
    for name, ts in kernel_parts.items():
        m = sum(ts) / len(ts)
        if m > dom_ms:
            dom_name, dom_ms = name, m
    # deliveries that are a single fused library call count as one kernel group
    for name, ts in per_delivery.items():
        if name.split("/")[0] in ("systematic", "stratified"):
            m = sum(ts) / len(ts)
            if m > dom_ms:
                dom_name, dom_ms = name, m
    alg, dt = dom_name.split("/")
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as fh:
            tr = json.load(fh)
        if n == N_DEFAULT and dom_name in tr:
            traffic = float(tr[dom_name]["bytes"])
    except Exception:
        pass
    s_bytes = 4 if dt == "f32" else 8
    alg_bytes = algorithmic_bytes(alg, s_bytes, n, trips[dt])
    achieved = alg_bytes / (dom_ms * 1e-3) / 1e9

    # ---------------- e2e: host buffers through the public API ----------------
    # Every delivery's weights come from pinned host memory and its ancestry
    # goes back to pinned host memory, inside the timed region.  The copies
    # run on two copy streams pipelined with the resampling kernels (later
    # deliveries' weights upload while earlier ones compute; results download
    # while later deliveries compute) -- the B200-native way to feed the API;
    # the device-only number is `value`.  The host link is the floor here:
    # the same uploads and downloads with no compute take ~1.4 ms per step
    # (H2D and D2H share the link; reported as `link_only_ms`).
    host_w = {dt: weights[dt].cpu().pin_memory() for dt in DTYPES}
    host_c = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in jobs]
    dev_w = [torch.empty_like(weights[dt]) for (_, _, _, dt) in jobs]
    dev_c = [torch.empty(n, dtype=torch.int32, device=dev) for _ in jobs]
    copy_stream = torch.cuda.Stream(device=dev)  # uploads
    down_stream = torch.cuda.Stream(device=dev)  # joins the downloads (the other copy direction)
    # one download stream per delivery: a result leaves as soon as its
    # delivery is done instead of queueing behind a longer one
    down_streams = [torch.cuda.Stream(device=dev) for _ in jobs]
    h2d = sum(host_w[dt].numel() * host_w[dt].element_size() for (_, _, _, dt) in jobs)
    d2h = len(jobs) * n * 4
    e2e_ms = 0.0
    # Schedule (measured on B200, N = 2^20): uploads take ~1.3 ms, the ten
    # deliveries ~1.2 ms of concurrent compute, downloads ~0.8 ms, so the
    # three must overlap.  The long deliveries (rejection, Metropolis) run
    # one after another on one compute stream, the short ones on a second,
    # and the upload order interleaves the two classes (f32 first: smaller
    # uploads start compute sooner) so results start downloading while
    # later weights still upload; the last upload (the smallest job) gets a
    # stream of its own so it never queues: 1.62 ms per step, against
    # 1.9-2.0 ms with every delivery on its own stream (longest upload
    # first) and 1.80 ms round-robin over two streams; stream priorities did
    # not help.
    names = [f"{jobs[k][1]}/{jobs[k][3]}" for k in range(len(jobs))]
    seq = os.environ.get("PFR_E2E_SEQ", "systematic/f32,rejection/f32,rejection/f64,stratified/f32,metropolis/f32,"
                         "metropolis/f64,multinomial/f32,stratified/f64,multinomial/f64,systematic/f64").split(",")
    order = [names.index(x) for x in seq]
    e2e_streams = [torch.cuda.Stream(device=dev) for _ in range(3)]
    stream_of = {k: e2e_streams[0 if jobs[k][1] in ("rejection", "metropolis") else 1] for k in order}
    stream_of[order[-1]] = e2e_streams[2]  # the last upload (the smallest job) never queues behind another
    if os.environ.get("PFR_E2E_STREAMS") == "each":  # A/B: every delivery on its own stream
        stream_of = {k: torch.cuda.Stream(device=dev) for k in order}

    for s in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda._sleep(STEP_PREROLL_CYCLES)
        copy_stream.wait_stream(stream)
        down_stream.wait_stream(stream)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(copy_stream)
        up = {}
        dbg = os.environ.get("PFR_BENCH_DEBUG") == "2"
        tl = {}
        for k in order:
            dt = jobs[k][3]
            with torch.cuda.stream(copy_stream):
                dev_w[k].copy_(host_w[dt], non_blocking=True)
                ev = torch.cuda.Event(enable_timing=dbg)
                ev.record(copy_stream)
            up[k] = ev
        for k in order:
            i, alg, j, dt = jobs[k]
            sk = stream_of[k]
            sk.wait_event(up[k])
            with torch.cuda.stream(sk):
                c = run_delivery(alg, dt, dev_w[k], pf.RngStream(50_000 + s, (rank, i, j)), dev_c[k])
                done = torch.cuda.Event(enable_timing=dbg)
                done.record(sk)
            dk = down_streams[k]
            c.record_stream(dk)
            dk.wait_event(done)
            with torch.cuda.stream(dk):
                host_c[k].copy_(c, non_blocking=True)
                if dbg:
                    fin = torch.cuda.Event(enable_timing=True)
                    fin.record(dk)
                    tl[k] = (up[k], done, fin)
        down_stream.wait_stream(copy_stream)
        for dk in down_streams:
            down_stream.wait_stream(dk)
        e1.record(down_stream)
        torch.cuda.synchronize()
        if os.environ.get("PFR_BENCH_DEBUG"):
            print(f"e2e step {s}: {e0.elapsed_time(e1):.3f} ms", file=sys.stderr, flush=True)
            for k in (order if dbg else []):
                u_, d_, f_ = tl[k]
                print(f"   {jobs[k][1]:12s}/{jobs[k][3]}: uploaded {e0.elapsed_time(u_):.3f} computed "
                      f"{e0.elapsed_time(d_):.3f} downloaded {e0.elapsed_time(f_):.3f}", file=sys.stderr, flush=True)
        if s >= args.warmup:
            e2e_ms += e0.elapsed_time(e1)
    # the link floor: the step's copies alone (uploads and downloads issued
    # together on two streams, no compute)
    link_ms = []
    down_only = torch.cuda.Stream(device=dev)
    for s in range(4):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record(copy_stream)
        down_only.wait_event(e0)
        with torch.cuda.stream(copy_stream):
            for k, (i, alg, j, dt) in enumerate(jobs):
                dev_w[k].copy_(host_w[dt], non_blocking=True)
        with torch.cuda.stream(down_only):
            for k in range(len(jobs)):
                host_c[k].copy_(dev_c[k], non_blocking=True)
        e1.record(copy_stream)
        e2.record(down_only)
        torch.cuda.synchronize()
        if s:
            link_ms.append(max(e0.elapsed_time(e1), e0.elapsed_time(e2)))
    link_only_ms = statistics.median(link_ms)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = world * units_per_step / (e2e_ms / args.steps * 1e-3)

    clk.__exit__(None, None, None)
    clocks = clk.summary((t_wall0, t_wall1))

    # ---------------- north-star targets: N = 2^24 float32 ----------------
    targets = None
    probes = None
    if rank == 0:
        try:
            probes = gather_probes(torch, dev, stream)
        except Exception as exc:  # optional measurement leg
            probes = {"error": f"{type(exc).__name__}: {exc}"[:200]}
    if not args.no_targets:
        targets = north_star_targets(pf, torch, dev, stream, flush, hbm, probes=probes) if rank == 0 else {}
        # config 4: ONE filter of N = 2^28 float32, weight-sharded over the ranks
        try:
            targets.update(c4_targets(pf, torch, dev, stream, flush, hbm, rank, world))
        except Exception as exc:  # keep the bench line even if this optional leg fails
            targets["c4_error"] = f"{type(exc).__name__}: {exc}"[:300]
        try:
            targets.update(c5_targets(pf, torch, dev, stream, rank, world))
        except Exception as exc:
            targets["c5_error"] = f"{type(exc).__name__}: {exc}"[:300]
        if rank == 0:
            try:
                targets.update(c3_targets(pf, torch, dev, stream))
            except Exception as exc:
                targets["c3_error"] = f"{type(exc).__name__}: {exc}"[:300]

    # ---------------- CPU baseline (rank 0, N=1 only) ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import multiprocessing as mp

        cores = min(os.cpu_count() or 1, len(ALGS) * len(DTYPES))
        with mp.get_context("spawn").Pool(cores) as pool:
            cpu_s = cpu_step(n, pool)
        cpu = {"value": units_per_step / cpu_s, "unit": "particles/s", "cores": cores, "kind": "port",
               "sample": f"one step (5 resamplers x f32/f64 at N=2^{int(math.log2(n))}) of the oracle port "
                         f"(NumPy + Python chain walk, like the reference), {cores} processes, {cpu_s:.1f} s",
               **host_cpu_info()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "particles/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32,f64 weights; f64 positions; int32 indices",
            "data": "synthetic i.i.d. log-normal weights (sigma=1), resident in HBM",
            "config": workload_config(n, world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "kernel": dom_name,
                         "algorithmic_bytes": alg_bytes, "kernel_ms": dom_ms, "peak_source": peak_src,
                         "traffic_source": "profiles/r02_traffic.json (ncu, per launch)",
                         "note": "algorithmic bytes count every proposal's weight gather (SURVEY 8(d)); the "
                                 "weights are L2 resident at N=2^20 and random gathers are bound by the L1TEX "
                                 "sector rate, not HBM; rejection skips the gathers whose outcome a shared-memory "
                                 "certain-reject table decides and is then bound by Philox issue (DESIGN.md 3.4)"},
            "sequential": {"ms_per_step": seq_ms_per_step, "value": seq_value, "gpu_launches": seq_launches,
                           "note": "the same ten deliveries one at a time, L2 flushed before each"},
            "gather_probes": probes,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "particles/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms / args.steps, "link_only_ms": link_only_ms,
                    "note": "pinned host buffers; uploads on one copy stream in an order interleaving long "
                            "and short deliveries, the long ones (rejection, Metropolis) computed in sequence on "
                            "one stream and the short ones on another, each result downloaded on its own stream "
                            "as soon as its delivery is done; link_only_ms = the same copies with no compute "
                            "(the host-link floor); results are int32 indices (the C ABI's output; the "
                            "reference's numpy arrays are int64 -- index_dtype=torch.int64 converts on the device "
                            "at twice the download bytes)"},
            "gpu_launches": launches,
            "clocks": clocks,
            "per_delivery_ms": {k: sum(v) / len(v) for k, v in per_delivery.items()},
            "status_bits": status,
            "targets": targets,
        }
        key = f"{dt}_2^{n.bit_length() - 1}"
        if alg in ("rejection", "metropolis") and probes and key in probes:
            gathers = (trips[dt] if alg == "rejection" else B_STEPS) * n
            g = gathers / (dom_ms * 1e-3) / 1e9
            peak = probes[key]["ggather_per_s"]
            line["roofline"]["gather_floor"] = {
                "achieved_ggather_per_s": g, "peak_ggather_per_s": peak, "frac": g / peak,
                "gathers_per_launch": gathers,
                "peak_source": f"pfr_probe_gather on the same-size ({key}) L2-resident vector, this run",
                "note": "gathers = proposals (trips) evaluated; frac > 1 means decided gathers were skipped "
                        "(rejection's certain-reject table)" if alg == "rejection" else "gathers = N x B steps"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def gather_probes(torch, dev, stream, reps=5):
    """Measured random-gather floor of the memory system (pfr_probe_gather:
    8 independent LCG streams per thread, 2 integer ops per gather): G
    gathers/s for L2-resident weight vectors (the N=2^20 headline and the
    2^24 north star) and for a 1 GiB vector (HBM random sectors, config 4)."""
    from paper_1301_4019_b200 import _lib as L

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    threads = sms * 8 * 256
    out = {}
    for name, log2n, eb in (("f32_2^20", 20, 4), ("f64_2^20", 20, 8), ("f32_2^24", 24, 4), ("f32_2^28", 28, 4)):
        n = 1 << log2n
        iters = max(1, (1 << 29) // (threads * 8))
        gathers = threads * 8 * iters
        buf = torch.randint(0, 2 ** 31 - 1, (n * eb // 4,), dtype=torch.int32, device=dev)
        sink = torch.zeros(1, dtype=torch.int64, device=dev)
        call = lambda: L.call("pfr_probe_gather", buf.data_ptr(), n, eb, gathers, sink.data_ptr(), stream.cuda_stream)
        call()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            call()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts)
        out[name] = {"ggather_per_s": gathers / (t * 1e-3) / 1e9, "bytes": n * eb}
        del buf, sink
    return out


def north_star_targets(pf, torch, dev, stream, flush, hbm, reps=10, probes=None):
    n = 1 << 24
    w = torch.from_numpy(log_normal_weights(n, 424242, np.float32)).to(dev)
    c = torch.empty(n, dtype=torch.int32, device=dev)
    a = torch.empty(n, dtype=torch.int32, device=dev)
    cfg = pf.ResamplerConfig("systematic")
    out = {}

    def timeit(fn):
        ts = []
        for r in range(reps + 3):
            flush.zero_()
            torch.cuda._sleep(PREROLL_CYCLES)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(r)
            e1.record(stream)
            torch.cuda.synchronize()
            if r >= 3:
                ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    t = timeit(lambda r: pf.deliver(w, cfg, pf.RngStream(r), index_dtype=torch.int32, out=c))
    b = (4 + 4) * n
    out["systematic_delivery_2^24_f32"] = {"us": t * 1e3, "particles_per_s": n / (t * 1e-3),
                                           "algorithmic_bytes": b, "achieved_gbs": b / (t * 1e-3) / 1e9,
                                           "frac": b / (t * 1e-3) / 1e9 / hbm, "target_frac": 0.70}
    # the same delivery from log-weights: fused (exp(lw - max) on load) vs
    # logweights_to_weights + deliver
    lw = torch.log(w)
    t_f = timeit(lambda r: pf.deliver(lw, cfg, pf.RngStream(r), index_dtype=torch.int32, out=c, log_weights=True))
    t_2 = timeit(lambda r: pf.deliver(pf.logweights_to_weights(lw), cfg, pf.RngStream(r), index_dtype=torch.int32,
                                      out=c))
    out["systematic_delivery_from_logweights_2^24_f32"] = {
        "us_fused": t_f * 1e3, "us_two_step": t_2 * 1e3, "particles_per_s": n / (t_f * 1e-3),
        "achieved_gbs": b / (t_f * 1e-3) / 1e9, "frac": b / (t_f * 1e-3) / 1e9 / hbm,
        "note": "algorithmic bytes s+4 as for weights; the fused path reads lw three times (max, K1, K2)"}
    del lw
    t = timeit(lambda r: pf.metropolis_ancestors(w, B_STEPS, pf.RngStream(r), index_dtype=torch.int32))
    b = (4 + 4 + B_STEPS * 4) * n
    out["metropolis_B32_2^24_f32_kernel"] = {"us": t * 1e3, "particles_per_s": n / (t * 1e-3),
                                             "algorithmic_bytes": b, "achieved_gbs": b / (t * 1e-3) / 1e9,
                                             "frac": b / (t * 1e-3) / 1e9 / hbm, "target_frac": 0.70}
    if probes and "f32_2^24" in probes:
        g = B_STEPS * n / (t * 1e-3) / 1e9
        peak = probes["f32_2^24"]["ggather_per_s"]
        out["metropolis_B32_2^24_f32_kernel"]["gather_floor"] = {
            "achieved_ggather_per_s": g, "peak_ggather_per_s": peak, "frac": g / peak,
            "peak_source": "pfr_probe_gather on a 64 MiB (L2-resident) vector, this run"}
    cfgm = pf.ResamplerConfig("metropolis", b=B_STEPS)
    t = timeit(lambda r: pf.deliver(w, cfgm, pf.RngStream(r), index_dtype=torch.int32))
    out["metropolis_B32_2^24_f32_delivery"] = {"us": t * 1e3, "particles_per_s": n / (t * 1e-3)}
    del w, c, a
    return out


def c4_targets(pf, torch, dev, stream, flush, hbm, rank, world, n_log2=28, reps=3):
    """BASELINE.json configs[3]: a single filter of N = 2^28 float32 log-normal
    weights, systematic delivery weight-sharded over `world` GPUs
    (paper_1301_4019_b200.sharded: shard totals all-gather + slot-word
    all-to-all + walker rounds, NCCL) and Metropolis(B=32) with the chains
    partitioned over the ranks.  At world == 1 this is the single-GPU path.
    Device time per rank (CUDA events), max over ranks."""
    import torch.distributed as dist

    from paper_1301_4019_b200 import sharded

    n = 1 << n_log2
    n_loc = n // world
    g = torch.Generator(device=dev)
    g.manual_seed(2828 + rank)
    lw = torch.randn(n_loc, device=dev, generator=g, dtype=torch.float32)
    mx = lw.max()
    if world > 1:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    w = torch.exp(lw - mx)
    del lw
    out = {}
    comm = sharded.DistComm() if world > 1 else None
    ops = sharded.CudaShardOps() if world > 1 else None

    def timed(fn):
        ts = []
        for r in range(reps + 1):
            flush.zero_()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            torch.cuda._sleep(PREROLL_CYCLES)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn(r)
            e1.record(stream)
            torch.cuda.synchronize()
            if r >= 1:
                ts.append(e0.elapsed_time(e1))
        t = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    cfg = pf.ResamplerConfig("systematic")
    if world == 1:
        c = torch.empty(n, dtype=torch.int32, device=dev)
        t = timed(lambda r: pf.deliver(w, cfg, pf.RngStream(r), index_dtype=torch.int32, out=c))
        del c
    else:
        t = timed(lambda r: sharded.deliver_sharded(w, cfg, pf.RngStream(r), comm=comm, ops=ops))
    b = 8 * n
    out[f"c4_systematic_delivery_2^{n_log2}_f32_{world}gpu"] = {
        "ms": t, "particles_per_s": n / (t * 1e-3), "algorithmic_bytes": b,
        "achieved_gbs_aggregate": b / (t * 1e-3) / 1e9, "frac_of_aggregate_hbm": b / (t * 1e-3) / 1e9 / (hbm * world),
        "scaling": "strong (one filter, fixed N)", "sharding": "weight shards, NCCL" if world > 1 else "single GPU"}
    if world == 1:
        t = timed(lambda r: pf.metropolis_ancestors(w, B_STEPS, pf.RngStream(r), index_dtype=torch.int32))
    else:
        t = timed(lambda r: sharded.metropolis_sharded(w, B_STEPS, pf.RngStream(r), comm=comm, ops=ops))
    b = (4 + 4 + B_STEPS * 4) * n
    out[f"c4_metropolis_B32_2^{n_log2}_f32_{world}gpu"] = {
        "ms": t, "particles_per_s": n / (t * 1e-3), "algorithmic_bytes": b,
        "achieved_gbs_aggregate": b / (t * 1e-3) / 1e9, "frac_of_aggregate_hbm": b / (t * 1e-3) / 1e9 / (hbm * world),
        "note": "gathers from a 1 GiB weight vector: HBM random-sector bound"}
    del w
    return out if rank == 0 else {}


def synthetic_observations(model, steps, filters, seed):
    """(filters, steps) observations simulated from the linear-Gaussian model
    with numpy's default generator (synthetic data; the bench does not need the
    reference's own draws)."""
    g = np.random.default_rng(seed)
    x = model.initial_mean + model.initial_std * g.standard_normal(filters)
    ys = np.empty((filters, steps))
    for t in range(steps):
        x = model.coeff * x + model.trans_std * g.standard_normal(filters)
        ys[:, t] = x + model.obs_std * g.standard_normal(filters)
    return ys


def c5_targets(pf, torch, dev, stream, rank, world, filters=4096, n_log2=16, steps=100):
    """BASELINE.json configs[4]: 4096 independent bootstrap filters x N = 2^16
    particles, T = 100, on the linear-Gaussian model; the filters are split
    over the ranks with no communication (each rank runs filters / world).
    Device time per rank, max over ranks."""
    import torch.distributed as dist

    from paper_1301_4019_b200.pf import LinearGaussianModel

    model = LinearGaussianModel(coeff=0.9, trans_std=1.0, obs_std=1.0)
    mine = filters // world
    ys = synthetic_observations(model, steps, mine, 1000 + rank * mine)
    n = 1 << n_log2
    pf.pf_run(model, ys[:, :3], n, seed=1)  # warm-up (allocations, module load)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    res = pf.pf_run(model, ys, n, "systematic", 0.5, seed=7)
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    resamples = int(res.resampled.sum()) * world
    return {f"c5_batched_pf_{filters}x2^{n_log2}_T{steps}_{world}gpu": {
        "ms": ms, "particle_steps_per_s": filters * n * steps / (ms * 1e-3),
        "particles_resampled_per_s": resamples * n / (ms * 1e-3), "resampling_events": resamples,
        "filters_per_gpu": mine, "note": "includes host->device copy of the observations and device->host "
                                         "copy of means/ESS/log-likelihood (the pf_run API call)",
        "cpu_reference_note": "SURVEY.md 6: the reference pf_run takes 1.95 s per filter (N=2^16, T=100) on "
                              "one core, i.e. ~2.2 core-hours for 4096 filters"}} if rank == 0 else {}


# the exact 1^T P^B oracle at N=2^22 (E[o_max]/(N p_max))
C3_EXACT_BIAS = {0.5: {1: .178, 4: .386, 16: .810, 32: .960, 64: .998, 256: 1.000},
                 1.0: {1: .016, 4: .040, 16: .128, 32: .234, 64: .408, 256: .875},
                 2.0: {1: .001, 4: .002, 16: .007, 32: .014, 64: .028, 256: .107}}


def c3_targets(pf, torch, dev, stream, n_log2=22, reps=8, sigmas=(0.5, 1.0, 1.5, 2.0, 3.0, 4.0),
               steps=(1, 4, 16, 32, 64, 256)):
    """BASELINE.json configs[2]: the log-weight sigma sweep at N = 2^22 f32.
    Metropolis bias vs B -- E[o_max]/(N p_max) over `reps` own-stream
    replicates (o_max: offspring of the heaviest particle), next to the exact
    1^T P^B values of SURVEY A.9 where the survey lists them -- and its
    recipe B (metropolis_num_steps, epsilon = p*/100); rejection acceptance
    N / sum(trips) against the analytic sum(w) / (N sup_w) with sup_w = max w
    = 1.  Device times are medians of CUDA events (no L2 flush: behaviour
    sweep, not a bandwidth number)."""
    n = 1 << n_log2
    out = {}

    def ev_time(fn):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return r, e0.elapsed_time(e1)

    for sigma in sigmas:
        g = np.random.default_rng(int(7000 + 100 * sigma))
        lw = g.normal(0.0, sigma, n)
        w64 = np.exp(lw - lw.max())
        w = torch.from_numpy(w64.astype(np.float32)).to(dev)
        wsum = float(w.double().sum())
        jmax = int(torch.argmax(w))
        p_max = float(w[jmax]) / wsum
        row = {"p_max": p_max, "ess_over_n": wsum ** 2 / float((w.double() ** 2).sum()) / n}
        bias = {}
        for b in steps:
            omax, ts = [], []
            for r in range(reps):
                a, t = ev_time(lambda: pf.metropolis_ancestors(w, b, pf.RngStream(r, (int(sigma * 10), b)),
                                                              index_dtype=torch.int32))
                omax.append(int((a == jmax).sum()))
                ts.append(t)
            m = float(np.mean(omax))
            se = float(np.std(omax, ddof=1) / math.sqrt(reps)) if reps > 1 else None
            cell = {"bias": m / (n * p_max), "bias_se": se / (n * p_max) if se is not None else None,
                    "kernel_ms": float(np.median(ts)), "ggather_per_s": b * n / (float(np.median(ts)) * 1e-3) / 1e9}
            ex = C3_EXACT_BIAS.get(sigma, {}).get(b)
            if ex is not None:
                cell["exact_survey"] = ex
            bias[str(b)] = cell
        row["metropolis"] = bias
        try:
            b_rec = int(pf.metropolis_num_steps(p_max, p_max / 100.0, n))
        except ValueError as exc:  # the recipe's own domain errors (resamplers.py:168-201)
            b_rec = None
            rec = {"error": str(exc)[:200]}
        if b_rec is not None:
            rec = {"B": b_rec}
        if b_rec is not None and b_rec * n <= (1 << 38):  # <= ~1 s per replicate
            omax, ts = [], []
            for r in range(2):
                a, t = ev_time(lambda: pf.metropolis_ancestors(w, b_rec, pf.RngStream(100 + r, (int(sigma * 10),)),
                                                              index_dtype=torch.int32))
                omax.append(int((a == jmax).sum()))
                ts.append(t)
            rec.update({"bias": float(np.mean(omax)) / (n * p_max), "kernel_ms": float(np.median(ts))})
        elif b_rec is not None:
            rec["skipped"] = "B * N above 2^38 gathers per replicate"
        row["metropolis_recipe"] = rec
        # rejection with the tight bound sup_w = max w = 1
        expected_trips = n / wsum
        m = n if expected_trips * n <= 2e11 else (1 << 16)  # huge sigma: a 2^16-slot sample
        wr = w if m == n else w[:m].contiguous()
        sup = float(wr.max())
        (a, trips), t = ev_time(lambda: pf.rejection_ancestors(wr, sup, pf.RngStream(9, (int(sigma * 10),)),
                                                               return_trips=True, max_rounds=10 ** 9,
                                                               index_dtype=torch.int32))
        tsum = float(trips.double().sum())
        row["rejection"] = {"acceptance": m / tsum, "analytic": float(wr.double().sum()) / (m * sup),
                            "mean_trips": tsum / m, "slots": m, "ms": t,
                            "gtrips_per_s": tsum / (t * 1e-3) / 1e9}
        out[f"sigma={sigma}"] = row
        del w, a
    return {f"c3_sigma_sweep_2^{n_log2}_f32": out}


if __name__ == "__main__":
    main()
