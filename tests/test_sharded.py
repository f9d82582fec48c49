"""The multi-GPU protocol of paper_1301_4019_b200.sharded.

CPU: the host protocol (shard totals, slot-word exchange, walker rounds across
shard boundaries, chain-partitioned Metropolis) with the NumPy stand-in ops,
over (a) G virtual ranks in threads and (b) real processes with the gloo
backend (world size 2), checked against the oracle's single-process delivery.
GPU: the same protocol with the CUDA kernels (virtual ranks on one B200),
checked against the single-GPU path and the oracle.

Weights are small integers stored as float64 so every partial sum is exact and
the sharded result must equal the reference bit for bit.
"""

from __future__ import annotations

import os
import socket
import threading

import numpy as np
import pytest
import torch

from oracle import pfr_oracle as orc
from paper_1301_4019_b200.resamplers import ResamplerConfig
from paper_1301_4019_b200.rng import RngStream
from paper_1301_4019_b200.sharded import ThreadComm, deliver_sharded

from .shard_ops_cpu import NumpyShardOps


def int_weights(n, seed, spread=50, zeros=0.2):
    g = np.random.default_rng(seed)
    w = g.integers(0, spread, n).astype(np.float64)
    w[g.random(n) < zeros] = 0.0
    w[0] += 1.0
    return w


def near_uniform_int_weights(n, seed):
    """weights 100 +- 10: almost every parent keeps one child, the slot/parent
    drift random-walks, and loser chains run for hundreds of steps across every
    shard boundary"""
    g = np.random.default_rng(seed)
    return (100 + g.integers(-10, 11, n)).astype(np.float64)


def split(n, world, seed):
    g = np.random.default_rng(seed)
    cuts = np.sort(g.choice(np.arange(1, n), world - 1, replace=False))
    return np.concatenate([[0], cuts, [n]])


def run_threads(world, fn):
    out = [None] * world
    err = []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001 -- re-raised in the caller
            err.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    if err:
        raise err[0]
    return out


def sharded_threads(w, world, alg, rs, ops_factory, cuts=None, **kw):
    cuts = split(w.size, world, 7) if cuts is None else cuts
    comms = ThreadComm.group(world)
    cfg = ResamplerConfig(alg, b=kw.pop("b", None))
    mode = kw.pop("rng_mode", "numpy")

    def fn(r):
        ops = ops_factory()
        shard = torch.from_numpy(w[cuts[r]: cuts[r + 1]].copy())
        return deliver_sharded(shard, cfg, rs, comm=comms[r], ops=ops, rng_mode=mode, return_max_steps=True, **kw)

    res = run_threads(world, fn)
    c = np.concatenate([x[0].cpu().numpy() for x in res]).astype(np.int64)
    return c, res[0][1]


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("alg", ["systematic", "stratified"])
def test_threads_offspring_equals_reference(world, alg):
    w = int_weights(1500, 11 + world)
    rs = RngStream(99, (world,))
    c, steps = sharded_threads(w, world, alg, rs, NumpyShardOps)
    want, want_steps = orc.permute(orc.expand_cumulative(
        orc.systematic(w, orc.systematic_offset(rs.seed, rs.ids)) if alg == "systematic"
        else orc.stratified(w, orc.stratified_uniforms(rs.seed, rs.ids, w.size))), with_steps=True)
    np.testing.assert_array_equal(c, want)
    assert orc.satisfies_predicate(c)
    if alg == "systematic":
        assert steps == want_steps


def test_threads_long_chains_cross_every_boundary():
    w = near_uniform_int_weights(3000, 5)
    rs = RngStream(3)
    cuts = np.array([0, 400, 401, 1700, 3000])  # includes a one-element shard
    c, steps = sharded_threads(w, 4, "systematic", rs, NumpyShardOps, cuts=cuts)
    want, want_steps = orc.permute(orc.expand_cumulative(orc.systematic(w, orc.systematic_offset(3, ()))),
                                   with_steps=True)
    np.testing.assert_array_equal(c, want)
    assert steps == want_steps and steps > 50


@pytest.mark.parametrize("alg", ["metropolis", "multinomial", "rejection"])
def test_threads_ancestry_algorithms(alg):
    w = int_weights(1024, 21)
    rs = RngStream(5, (1,))
    c, _ = sharded_threads(w, 3, alg, rs, NumpyShardOps, b=8 if alg == "metropolis" else None)
    want = orc.deliver(w, alg, rs.seed, rs.ids, b=8)
    np.testing.assert_array_equal(c, want)


def test_threads_rejection_slots_partitioned():
    """Rejection partitions the output slots over the all-gathered weights
    (SURVEY 8(e)); the CPU stand-in slices the reference loop."""
    w = int_weights(1024, 33)
    rs = RngStream(8, (2,))
    c, _ = sharded_threads(w, 3, "rejection", rs, NumpyShardOps)
    a = orc.rejection_stream(w, float(w.max()), rs.seed, rs.ids)[0]
    np.testing.assert_array_equal(c, orc.permute(a))


def test_threads_v2_and_general_protocols():
    """the default halo keeps i.i.d. weights on protocol v2; a zero halo
    forces every rank onto the general protocol together -- same result"""
    from paper_1301_4019_b200 import sharded

    w = int_weights(3000, 17)
    rs = RngStream(2)
    want = orc.deliver(w, "systematic", rs.seed, rs.ids)
    before = dict(sharded.protocol_counts)
    c, _ = sharded_threads(w, 3, "systematic", rs, NumpyShardOps)
    np.testing.assert_array_equal(c, want)
    assert sharded.protocol_counts["v2"] == before["v2"] + 3
    os.environ["PFR_SHARD_HALO"] = "0"
    try:
        c, _ = sharded_threads(w, 3, "systematic", rs, NumpyShardOps)
    finally:
        del os.environ["PFR_SHARD_HALO"]
    np.testing.assert_array_equal(c, want)
    assert sharded.protocol_counts["general"] == before["general"] + 3


def test_threads_errors_raise_on_every_rank():
    w = int_weights(300, 2)
    w[250] = -1.0
    with pytest.raises(ValueError, match="non-negative"):
        sharded_threads(w, 2, "systematic", RngStream(1), NumpyShardOps)


# ---------------------------------------------------------------------------
# real processes, gloo backend


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, alg, n, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1301_4019_b200.sharded import DistComm

        comm = DistComm()
        w = near_uniform_int_weights(n, 8) if alg == "systematic-long" else int_weights(n, 8)
        algorithm = "systematic" if alg == "systematic-long" else alg
        cuts = split(n, world, 3)
        rs = RngStream(42, (7,))
        shard = torch.from_numpy(w[cuts[rank]: cuts[rank + 1]].copy())
        cfg = ResamplerConfig(algorithm, b=6 if algorithm == "metropolis" else None)
        c, steps = deliver_sharded(shard, cfg, rs, comm=comm, ops=NumpyShardOps(), rng_mode="numpy",
                                   return_max_steps=True)
        full = comm.all_gather_var(c).numpy().astype(np.int64)
        want = orc.deliver(w, algorithm, rs.seed, rs.ids, b=6)
        ok = bool(np.array_equal(full, want)) and orc.satisfies_predicate(full)
        q.put((rank, ok, int(steps) if steps is not None else -1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("alg", ["systematic", "systematic-long", "stratified", "metropolis", "multinomial",
                                 "rejection"])
def test_gloo_world2(alg):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, alg, 2000, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert all(ok for _, ok, _ in res), res


# ---------------------------------------------------------------------------
# GPU: CUDA kernels, virtual ranks on one device


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("alg", ["systematic", "stratified"])
def test_gpu_sharded_offspring_matches_reference(world, alg):
    from paper_1301_4019_b200.sharded import CudaShardOps

    w = int_weights(1 << 16, 30 + world)
    rs = RngStream(17, (world,))
    c, steps = sharded_threads(w, world, alg, rs, CudaShardOps)
    want = orc.deliver(w, alg, rs.seed, rs.ids)
    np.testing.assert_array_equal(c, want)


@pytest.mark.gpu
def test_gpu_sharded_long_chains():
    from paper_1301_4019_b200.sharded import CudaShardOps

    w = near_uniform_int_weights(20000, 9)
    rs = RngStream(4)
    c, steps = sharded_threads(w, 4, "systematic", rs, CudaShardOps)
    want, want_steps = orc.permute(orc.expand_cumulative(orc.systematic(w, orc.systematic_offset(4, ()))),
                                   with_steps=True)
    np.testing.assert_array_equal(c, want)
    assert steps == want_steps


@pytest.mark.gpu
def test_gpu_sharded_lognormal_vs_single_gpu():
    """float64 log-normal weights at 2^20 over 8 virtual ranks: equal to the
    single-GPU delivery outside the rounding-fragile set (expected empty)."""
    import paper_1301_4019_b200 as pf
    from paper_1301_4019_b200.sharded import CudaShardOps

    g = np.random.default_rng(12)
    lw = g.normal(0, 1, 1 << 20)
    w = np.exp(lw - lw.max())
    rs = RngStream(8)
    c, _ = sharded_threads(w, 8, "systematic", rs, CudaShardOps, cuts=np.linspace(0, w.size, 9).astype(np.int64))
    single = pf.deliver(w, ResamplerConfig("systematic"), rs, rng_mode="numpy").cpu().numpy()
    assert orc.satisfies_predicate(c)
    assert np.array_equal(np.bincount(c, minlength=w.size), np.bincount(single, minlength=w.size))
    np.testing.assert_array_equal(c, single)


@pytest.mark.gpu
def test_gpu_sharded_metropolis_bit_identical():
    import paper_1301_4019_b200 as pf
    from paper_1301_4019_b200.sharded import CudaShardOps

    g = np.random.default_rng(3)
    lw = g.normal(0, 1, 1 << 16)
    w = np.exp(lw - lw.max()).astype(np.float32)
    rs = RngStream(11)
    c, _ = sharded_threads(w, 4, "metropolis", rs, CudaShardOps, b=32)
    single = pf.deliver(w, ResamplerConfig("metropolis", b=32), rs, rng_mode="numpy").cpu().numpy()
    np.testing.assert_array_equal(c, single)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_gpu_sharded_rejection_bit_identical(world):
    """Slot-partitioned rejection (pfr_rejection_range on each rank's slots,
    every slot on its global Philox stream) equals the single-GPU delivery."""
    import paper_1301_4019_b200 as pf
    from paper_1301_4019_b200.sharded import CudaShardOps

    g = np.random.default_rng(5)
    lw = g.normal(0, 1, 1 << 16)
    w = np.exp(lw - lw.max()).astype(np.float32)
    rs = RngStream(12, (world,))
    c, _ = sharded_threads(w, world, "rejection", rs, CudaShardOps, rng_mode="philox")
    single = pf.deliver(w, ResamplerConfig("rejection"), rs, rng_mode="philox").cpu().numpy()
    np.testing.assert_array_equal(c, single)


@pytest.mark.gpu
@pytest.mark.parametrize("procs", [2, 3])
def test_gpu_sharded_real_processes(procs):
    """torch.distributed with real processes (gloo; every rank's kernels on
    one GPU, uneven shards at 3): systematic, stratified, Metropolis,
    rejection (plain and capped) and (replicated) multinomial deliveries
    equal the single-GPU ones."""
    import subprocess
    import sys

    port = 29600 + procs
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={procs}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(os.path.dirname(__file__), "shard_gloo_worker.py"), "18"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert r.stdout.count("identical") == 6 and "DIFFERENT" not in r.stdout, r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("mode", ["philox", "numpy"])
def test_gpu_sharded_multinomial_bit_identical(world, mode):
    """Slot-partitioned multinomial (pfr_multinomial_range: every rank merges
    only its slots' sorted uniforms with W) plus the partitioned permute
    (pfr_permute_range) equal the single-GPU delivery at 2/4/8 virtual ranks."""
    import paper_1301_4019_b200 as pf
    from paper_1301_4019_b200.sharded import CudaShardOps

    g = np.random.default_rng(40 + world)
    lw = g.normal(0, 1, 1 << 16)
    w = np.exp(lw - lw.max())
    rs = RngStream(21, (world,))
    cuts = split(w.size, world, 5)
    c, steps = sharded_threads(w, world, "multinomial", rs, CudaShardOps, cuts=cuts, rng_mode=mode)
    single, want_steps = pf.deliver(w, ResamplerConfig("multinomial"), rs, rng_mode=mode, return_max_steps=True)
    np.testing.assert_array_equal(c, single.cpu().numpy())
    assert steps == int(want_steps)


@pytest.mark.gpu
def test_gpu_permute_range_union_is_the_permute():
    """pfr_permute_range over any index partition reproduces permute_parallel,
    including its longest chain (random ancestries and an adversarial chain)."""
    import paper_1301_4019_b200 as pf
    from paper_1301_4019_b200.sharded import CudaShardOps

    g = np.random.default_rng(2)
    n = 4000  # the adversarial chain (n - 2 hops) stays under the 4096-hop walk bound
    cases = [g.integers(0, n, n), np.sort(g.integers(0, n, n)), np.r_[np.arange(1, n), [n - 1]]]
    ops = CudaShardOps()
    long_chain = np.r_[np.arange(1, 6000), [5999]].astype(np.int32)
    _, _, flag = ops.permute_range(torch.from_numpy(long_chain), 0, 6000)
    assert ops.overflowed(flag)  # beyond the bound: the caller falls back to the full permute
    for a in cases:
        want, want_steps = orc.permute(a, with_steps=True)
        cuts = [0, 1, 1234, 2500, n]  # uneven, with a one-index part
        parts, steps = [], 0
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            c, st, flag = ops.permute_range(torch.from_numpy(a.astype(np.int32)), lo, hi - lo)
            assert not ops.overflowed(flag)
            parts.append(c.cpu().numpy())
            steps = max(steps, int(st.item()))
        np.testing.assert_array_equal(np.concatenate(parts), want)
        assert steps == want_steps
        ops.check()


@pytest.mark.gpu
def test_gpu_sharded_zero_weight_shard():
    """A rank whose whole shard weighs zero has an empty slot window (ADVICE:
    it must not fail alone while the others wait in the next collective)."""
    import paper_1301_4019_b200 as pf
    from paper_1301_4019_b200.sharded import CudaShardOps

    w = int_weights(6000, 3, zeros=0.0)
    w[2000:4000] = 0.0
    rs = RngStream(6)
    for alg in ("systematic", "stratified"):
        c, _ = sharded_threads(w, 3, alg, rs, CudaShardOps, cuts=np.array([0, 2000, 4000, 6000]))
        want = orc.deliver(w, alg, rs.seed, rs.ids)
        np.testing.assert_array_equal(c, want)


@pytest.mark.gpu
@pytest.mark.parametrize("alg", ["metropolis", "rejection", "multinomial"])
def test_gpu_sharded_bad_weights_raise_on_every_rank(alg):
    """Negative weights on one shard raise the reference's ValueError on every
    rank (the validation bits travel with the shard sizes)."""
    from paper_1301_4019_b200.sharded import CudaShardOps

    w = int_weights(3000, 4)
    w[2500] = -1.0
    mode = "philox" if alg == "rejection" else "numpy"
    with pytest.raises(ValueError, match="non-negative"):
        sharded_threads(w, 2, alg, RngStream(3), CudaShardOps, b=8 if alg == "metropolis" else None, rng_mode=mode)
