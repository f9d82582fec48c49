"""One resampling problem spread over several GPUs.

The reference has no distributed path; its single-process
semantics (resamplers.py:105-153, 204-234; ancestry.py:139-174) are kept
exactly, and the data is partitioned so that each GPU streams only its share:

* **systematic / stratified, one weight-sharded filter** -- rank g holds the
  contiguous weight shard [base_g, base_g + n_g).  It scans its shard locally
  (float64), an all-gather of the G shard totals gives every rank the weight
  before its shard and W_N, and each rank computes the cumulative offspring
  of its own parents in GLOBAL slot numbers (pfr_shard_offspring).  The slot
  words of those parents (parent | FIRST) go, by one all-to-all, to the ranks
  that own the slot indices; each rank then resolves the in-place ancestry
  of its indices (pfr_shard_resolve).  Loser chains that cross a shard
  boundary continue as walkers (hole, slot, steps) routed to the owner of
  `slot` (pfr_shard_advance) until they reach their loser, and the value goes
  back to the owner of the hole.  Drift between slot and parent is ~sqrt(N),
  so only a thin band at each boundary travels.
* **Metropolis / rejection / multinomial** -- the weight vector is
  all-gathered once (the shard sizes and validation bits travel in one
  all-gather before it, so every rank raises together); rank g draws the
  ancestors of its output slots with their global stream numbers
  (pfr_metropolis_range, pfr_rejection_range, pfr_multinomial_range: the
  union is bit-identical to the single-GPU result).  The ancestry is
  all-gathered once more and every rank resolves the in-place ancestry of its
  OWN indices only (pfr_permute_range: claims over the full ancestry, loser
  chains walked backwards from the rank's holes); a chain past the walk
  bound on any rank falls back to the replicated permute.
* **batched independent filters** need no communication at all (each rank
  calls the single-GPU API on its own filters).

Collectives go through a small `Comm` interface: `DistComm` wraps
torch.distributed (NCCL on B200s, gloo for CPU tests); `ThreadComm` runs G
virtual ranks as threads of one process (one GPU), which is how the GPU tests
exercise the sharded path on a single device.  The per-rank compute goes
through `CudaShardOps` (libpfr kernels); there is no CPU implementation in
the product.
"""

from __future__ import annotations

import math
import os
import threading

import numpy as np
import torch

from . import _lib as L
from .rng import as_stream

__all__ = ["DistComm", "ThreadComm", "CudaShardOps", "deliver_sharded", "metropolis_sharded", "shard_bounds"]

_FIRST = 0x80000000
_TAG_SYSTEMATIC = 0x5359


# ---------------------------------------------------------------------------
# collectives


class DistComm:
    """torch.distributed collectives on `group` (payload tensors live on `device`:
    CUDA for NCCL, CPU for gloo)."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
                else torch.device("cpu")
        self.device = torch.device(device)

    def all_gather_scalars(self, x, dtype) -> list:
        t = torch.tensor([x], dtype=dtype, device=self.device)
        out = torch.empty(self.world, dtype=dtype, device=self.device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().tolist()

    def all_to_all(self, send: torch.Tensor, send_counts: list[int], width: int = 1) -> torch.Tensor:
        """Variable all-to-all of rows of `width` int32; returns received rows in rank order."""
        sc = torch.tensor(send_counts, dtype=torch.int64, device=self.device)
        rc = torch.empty_like(sc)
        self.dist.all_to_all_single(rc, sc, group=self.group)
        recv_counts = rc.cpu().tolist()
        flat = send.reshape(-1).to(self.device)
        out = torch.empty(sum(recv_counts) * width, dtype=send.dtype, device=self.device)
        self.dist.all_to_all_single(out, flat, [c * width for c in recv_counts], [c * width for c in send_counts],
                                    group=self.group)
        return out.reshape(-1, width) if width > 1 else out

    def all_gather_fixed(self, t: torch.Tensor) -> torch.Tensor:
        """all-gather of equal-size tensors, rank order, staying on the
        communicator's device (NCCL: no host round trip)"""
        t = t.reshape(-1).to(self.device)
        out = torch.empty(self.world * t.numel(), dtype=t.dtype, device=self.device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return out

    def neighbor_exchange(self, to_left: torch.Tensor, to_right: torch.Tensor):
        """send to_left to rank-1 and to_right to rank+1 (equal sizes), receive
        (from_left, from_right) -- None at the ends; point to point (NCCL:
        device to device, no host round trip)"""
        reqs, ops = [], []
        from_left = from_right = None
        P2P = self.dist.P2POp
        if self.rank > 0:
            from_left = torch.empty_like(to_right, device=self.device)
            ops += [P2P(self.dist.isend, to_left.contiguous().to(self.device), self.rank - 1, self.group),
                    P2P(self.dist.irecv, from_left, self.rank - 1, self.group)]
        if self.rank + 1 < self.world:
            from_right = torch.empty_like(to_left, device=self.device)
            ops += [P2P(self.dist.isend, to_right.contiguous().to(self.device), self.rank + 1, self.group),
                    P2P(self.dist.irecv, from_right, self.rank + 1, self.group)]
        if ops:
            reqs = self.dist.batch_isend_irecv(ops)
        for r in reqs:
            r.wait()
        return from_left, from_right

    def all_gather_var(self, t: torch.Tensor) -> torch.Tensor:
        sizes = [int(s) for s in self.all_gather_scalars(t.numel(), torch.int64)]
        m = max(sizes)
        pad = torch.zeros(m, dtype=t.dtype, device=self.device)
        pad[: t.numel()] = t.to(self.device)
        out = torch.empty(m * self.world, dtype=t.dtype, device=self.device)
        self.dist.all_gather_into_tensor(out, pad, group=self.group)
        return torch.cat([out[r * m: r * m + sizes[r]] for r in range(self.world)])


class _ThreadHub:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world


class ThreadComm:
    """G virtual ranks as threads of one process (shared device memory); the
    collectives exchange references under a barrier.  Create one hub per
    group with `ThreadComm.group(G)` and give thread g `comms[g]`."""

    def __init__(self, hub: _ThreadHub, rank: int, device=None):
        self.hub = hub
        self.rank = rank
        self.world = hub.world
        self.device = torch.device(device) if device is not None else None  # None: tensors stay where they are
        # every virtual rank enqueues on its own CUDA stream, as a real rank
        # does on its own GPU: host threads interleaving launches on ONE
        # stream measured unsafe (a thread stress test: 3 of 20 runs wrong)
        self.stream = torch.cuda.Stream() if torch.cuda.is_available() else None

    @staticmethod
    def group(world: int, device=None) -> list["ThreadComm"]:
        hub = _ThreadHub(world)
        return [ThreadComm(hub, r, device) for r in range(world)]

    def _exchange(self, obj, consume=lambda got: got):
        """publish obj, let `consume` read every rank's object, and only then
        release the peers: a producer must not free (and its allocator reuse)
        a tensor before every consumer's copy of it has run, so the copies
        are synchronised before the last barrier"""
        h = self.hub
        h.barrier.wait()
        h.slots[self.rank] = obj
        h.barrier.wait()
        out = consume(list(h.slots))
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.current_stream().synchronize()
        h.barrier.wait()
        return out

    def all_gather_scalars(self, x, dtype) -> list:
        return [type(x)(v) if not isinstance(x, torch.Tensor) else v for v in self._exchange(x)]

    def all_to_all(self, send: torch.Tensor, send_counts: list[int], width: int = 1) -> torch.Tensor:
        rows = send.reshape(-1, width) if width > 1 else send.reshape(-1)
        starts = np.concatenate([[0], np.cumsum(send_counts)]).astype(np.int64)
        pieces = [rows[starts[r]: starts[r + 1]] for r in range(self.world)]
        if rows.is_cuda:
            torch.cuda.current_stream().synchronize()  # producers' kernels done before peers read
        dev = self.device or send.device
        return self._exchange(pieces, lambda got: torch.cat([got[q][self.rank].to(dev) for q in range(self.world)]))

    def all_gather_fixed(self, t: torch.Tensor) -> torch.Tensor:
        return self.all_gather_var(t.reshape(-1))

    def neighbor_exchange(self, to_left: torch.Tensor, to_right: torch.Tensor):
        if to_left.is_cuda:
            torch.cuda.current_stream().synchronize()
        dev = self.device or to_left.device

        def pick(got):
            left = got[self.rank - 1][1].to(dev).clone() if self.rank > 0 else None
            right = got[self.rank + 1][0].to(dev).clone() if self.rank + 1 < self.world else None
            return left, right

        return self._exchange((to_left, to_right), pick)

    def all_gather_var(self, t: torch.Tensor) -> torch.Tensor:
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        dev = self.device or t.device
        return self._exchange(t, lambda got: torch.cat([g.to(dev) for g in got]))


# ---------------------------------------------------------------------------
# per-rank compute on the GPU (libpfr)


class CudaShardOps:
    """The per-rank kernels of the sharded path (include/pfr.h, 'weight-sharded').
    Owns its workspace and status word, so virtual ranks sharing a device do
    not share scratch."""

    def __init__(self):
        self.dev = L.device()
        self._ws = None
        self.status = torch.zeros(1, dtype=torch.int32, device=self.dev)

    def _workspace(self, n):
        need = int(L.lib().pfr_workspace_bytes(L.OP_ANY, int(n), 0))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=self.dev)
        return self._ws.data_ptr(), self._ws.numel()

    def tensor(self, x, dtype):
        return torch.as_tensor(x, dtype=dtype).to(self.dev)

    def _on_dev(self, t):
        """Protocol payloads arrive on the communicator's device (host memory
        for gloo): the kernels need them on this rank's GPU."""
        return torch.as_tensor(t).to(self.dev).contiguous()

    def status_bits(self) -> int:
        return L.read_status(self.status)

    def reset(self):
        """a fresh status word for this call (an earlier call's error bits
        must not leak into this one)"""
        self.status.zero_()

    def check_local(self, w_local):
        """check_weights (diagnostics.py:38-51) on this rank's shard, into the status word"""
        w = L.as_weights(w_local)
        L.call("pfr_check_weights", w.data_ptr(), w.numel(), L.dtype_code(w), self.status.data_ptr(),
               L.stream_handle())

    def check(self):
        bits = L.read_status(self.status)
        L.raise_weight_errors(bits & ~L.ST_POSITIVE, "w", False)
        if bits & L.ST_NOPROGRESS:
            from .resamplers import MAX_REJECTION_ROUNDS

            raise RuntimeError(f"rejection resampling made no progress after {MAX_REJECTION_ROUNDS} rounds; "
                               "the weight bound is far above every weight")
        if bits & L.ST_NONTERMINATION:
            raise RuntimeError("permutation chain walk failed to terminate")
        if bits & (L.ST_RANGE | L.ST_NOTMONOTONE):
            raise RuntimeError(f"sharded resampling: inconsistent shard data (status {bits:#x})")

    def local_scan(self, w: torch.Tensor):
        w = L.as_weights(w)
        n = w.numel()
        W = torch.empty(n, dtype=torch.float64, device=self.dev)
        ws, wsb = self._workspace(n)
        L.call("pfr_check_weights", w.data_ptr(), n, L.dtype_code(w), self.status.data_ptr(), L.stream_handle())
        L.call("pfr_scan", w.data_ptr(), W.data_ptr(), n, L.dtype_code(w), L.F64, L.ACC_F64 | L.SCAN_MONOTONE, 0, None,
               self.status.data_ptr(), ws, wsb, L.stream_handle())
        return W, float(W[-1].item())

    def systematic_offset(self, rng, mode):
        k0, k1 = as_stream(rng).key()
        r = L.PfrRng(k0, k1, L.rng_mode_code(mode), 0)
        return float(L.lib().pfr_stream_uniform(r, 0, _TAG_SYSTEMATIC))

    def offspring(self, W, wdtype, prefix, total, n_global, last, stratified, offset, uniforms, rng, mode):
        W = self._on_dev(W)
        n = W.numel()
        O = torch.empty(n, dtype=torch.int32, device=self.dev)
        k0, k1 = as_stream(rng).key() if rng is not None else (0, 0)
        r = L.PfrRng(k0, k1, L.rng_mode_code(mode), 0)
        uni = None if uniforms is None else torch.as_tensor(uniforms, dtype=torch.float64).to(self.dev).contiguous()
        L.call("pfr_shard_offspring", W.data_ptr(), n, L.F32 if wdtype == torch.float32 else L.F64, float(prefix),
               float(total), int(n_global), int(last), int(stratified), float(offset), L.ptr(uni), r, O.data_ptr(),
               L.stream_handle())
        return O

    def words(self, O, base, o_begin):
        O = self._on_dev(O)
        n = O.numel()
        o_end = int(O[-1].item())
        # a shard without offspring has an empty slot window: keep a 1-element
        # buffer (a null pointer is an argument error, and that rank would
        # raise alone while the others wait in the next collective)
        size = max(o_end - o_begin, 0)
        words = torch.empty(max(size, 1), dtype=torch.int32, device=self.dev)
        has = torch.empty(n, dtype=torch.uint8, device=self.dev)
        L.call("pfr_shard_words", O.data_ptr(), n, int(base), int(o_begin), words.data_ptr(), has.data_ptr(),
               self.status.data_ptr(), L.stream_handle())
        return words[:size], has

    def resolve(self, words, has, base):
        words, has = self._on_dev(words), self._on_dev(has)
        n = has.numel()
        c = torch.empty(n, dtype=torch.int32, device=self.dev)
        pend = torch.empty((n, 3), dtype=torch.int32, device=self.dev)
        cnt = torch.zeros(2, dtype=torch.int32, device=self.dev)  # [pending, max steps]
        L.call("pfr_shard_resolve", words.data_ptr(), has.data_ptr(), n, int(base), c.data_ptr(), pend.data_ptr(),
               cnt.data_ptr(), cnt[1:].data_ptr(), self.status.data_ptr(), L.stream_handle())
        k, steps = cnt.tolist()
        return c, pend[:k], steps

    def advance(self, walkers, words, base, n_loc):
        k = walkers.shape[0]
        done = torch.empty((max(k, 1), 2), dtype=torch.int32, device=self.dev)
        fwd = torch.empty((max(k, 1), 3), dtype=torch.int32, device=self.dev)
        cnt = torch.zeros(3, dtype=torch.int32, device=self.dev)  # [done, fwd, max steps]
        if k:
            walkers, words = self._on_dev(walkers), self._on_dev(words)
            L.call("pfr_shard_advance", walkers.data_ptr(), k, words.data_ptr(), int(n_loc), int(base),
                   done.data_ptr(), cnt[0:].data_ptr(), fwd.data_ptr(), cnt[1:].data_ptr(), cnt[2:].data_ptr(),
                   self.status.data_ptr(), L.stream_handle())
        nd, nf, steps = cnt.tolist()
        return done[:nd], fwd[:nf], steps

    def scatter(self, done, base, c):
        k = done.shape[0]
        if k:
            done = self._on_dev(done)
            L.call("pfr_shard_scatter", done.data_ptr(), k, int(base), c.numel(), c.data_ptr(),
                   self.status.data_ptr(), L.stream_handle())

    # ---- protocol v3: the shard's local work through the single-GPU kernels ----
    def local_end(self, w: torch.Tensor) -> torch.Tensor:
        """K1 over the shard (check_weights' flags into the status word) and the
        shard's END value (W at its last element in the delivery's
        association) as a 1-element device tensor"""
        w = L.as_weights(w)
        n = w.numel()
        end = torch.empty(1, dtype=torch.float64, device=self.dev)
        ws, wsb = self._workspace(n)
        L.call("pfr_shard_local_end", w.data_ptr(), n, L.dtype_code(w), end.data_ptr(), self.status.data_ptr(), ws, wsb,
               L.stream_handle())
        return end

    def shard_produce(self, w, base, n_global, pt, first, last, stratified, offset, uniforms, rng, mode, ext, slot_lo,
                      slot_hi):
        w = L.as_weights(w)
        n = w.numel()
        k0, k1 = as_stream(rng).key() if rng is not None else (0, 0)
        r = L.PfrRng(k0, k1, L.rng_mode_code(mode), 0)
        uni = None if uniforms is None else torch.as_tensor(uniforms, dtype=torch.float64).to(self.dev).contiguous()
        pt = self._on_dev(pt)
        ws, wsb = self._workspace(n)
        L.call("pfr_shard_produce", w.data_ptr(), n, L.dtype_code(w), int(base), int(n_global), pt.data_ptr(),
               int(first), int(last), int(stratified), float(offset), L.ptr(uni), r, ext.data_ptr(), int(slot_lo),
               int(slot_hi), self.status.data_ptr(), ws, wsb, L.stream_handle())

    def shard_resolve_fast(self, ext, slot_lo, slot_hi, base, n_loc, wdtype):
        c = torch.empty(n_loc, dtype=torch.int32, device=self.dev)
        st = torch.zeros(1, dtype=torch.int32, device=self.dev)
        ws, wsb = self._workspace(n_loc)
        L.call("pfr_shard_resolve_fast", int(n_loc), L.F32 if wdtype == torch.float32 else L.F64, int(base),
               ext.data_ptr(), int(slot_lo), int(slot_hi), c.data_ptr(), st.data_ptr(), self.status.data_ptr(), ws, wsb,
               L.stream_handle())
        return c, st

    def prefix_total(self, totals: torch.Tensor, rank: int) -> torch.Tensor:
        """{weight before this shard, W_N}: left folds of the shard END values
        in rank order (the same IEEE additions on every rank), on the device"""
        totals = self._on_dev(totals).to(torch.float64)
        acc = torch.zeros(1, dtype=torch.float64, device=self.dev)
        prefix = acc
        for r in range(totals.numel()):
            if r == rank:
                prefix = acc.clone()
            acc = acc + totals[r: r + 1]
        return torch.cat([prefix, acc])

    @staticmethod
    def bands(ext, n_loc, halo):
        """(this rank's ext[0, 2H), ext[n, n + 2H)): what the left and the
        right neighbour need"""
        return ext[: 2 * halo], ext[n_loc: n_loc + 2 * halo]

    def merge(self, ext, n_loc, halo, from_left, from_right):
        fl = None if from_left is None else self._on_dev(from_left)
        fr = None if from_right is None else self._on_dev(from_right)
        L.call("pfr_shard_merge_bands", ext.data_ptr(), int(n_loc), int(halo), L.ptr(fl), L.ptr(fr),
               L.stream_handle())

    def metropolis_range(self, w_full, b, rng, mode, c_begin, c_count):
        w_full = L.as_weights(w_full)
        a = torch.empty(c_count, dtype=torch.int32, device=self.dev)
        k0, k1 = as_stream(rng).key()
        r = L.PfrRng(k0, k1, L.rng_mode_code(mode), 0)
        L.call("pfr_metropolis_range", w_full.data_ptr(), w_full.numel(), L.dtype_code(w_full), int(b), r,
               int(c_begin), int(c_count), a.data_ptr(), self.status.data_ptr(), L.stream_handle())
        return a

    def rejection_range(self, w_full, config, rng, mode, s_begin, s_count):
        """rejection_ancestors(_capped) for slots [s_begin, s_begin + s_count)
        of the full weight vector (resamplers.py:237-310), global parent
        numbers; PHILOX stream only (like the single-GPU rejection)."""
        from .resamplers import MAX_REJECTION_ROUNDS

        if mode not in (None, "philox"):
            raise NotImplementedError("sharded rejection uses the GPU's own Philox stream")
        w_full = L.as_weights(w_full)
        capped = config.algorithm == "rejection-capped"
        if capped and config.sup_v is None:
            raise ValueError("rejection-capped requires sup_v")
        sup = config.sup_w if config.sup_w is not None else float(w_full.max())  # as resample_ancestors
        bound = float(config.sup_v if capped else sup)
        a = torch.empty(max(s_count, 1), dtype=torch.int32, device=self.dev)
        out_w = torch.empty(max(s_count, 1), dtype=w_full.dtype, device=self.dev) if capped else None
        k0, k1 = as_stream(rng).key()
        r = L.PfrRng(k0, k1, L.RNG_PHILOX, 0)
        ws, wsb = self._workspace(w_full.numel())
        L.call("pfr_rejection_range", w_full.data_ptr(), w_full.numel(), L.dtype_code(w_full),
               0.0 if capped else bound, bound if capped else 0.0, r, int(MAX_REJECTION_ROUNDS), int(s_begin),
               int(s_count), a.data_ptr(), None, L.ptr(out_w), self.status.data_ptr(), ws, wsb,
               L.stream_handle())
        return a[:s_count]

    def multinomial_range(self, w_full, rng, mode, s_begin, s_count, uniforms=None):
        """multinomial_ancestors (resamplers.py:56-74) for slots [s_begin,
        s_begin + s_count) of the full weight vector, global parent numbers."""
        w_full = L.as_weights(w_full)
        n = w_full.numel()
        a = torch.empty(max(s_count, 1), dtype=torch.int32, device=self.dev)
        k0, k1 = as_stream(rng).key() if rng is not None else (0, 0)
        r = L.PfrRng(k0, k1, L.rng_mode_code(mode), 0)
        uni = None if uniforms is None else torch.as_tensor(uniforms, dtype=torch.float64).to(self.dev).contiguous()
        ws, wsb = self._workspace(n)
        L.call("pfr_multinomial_range", w_full.data_ptr(), n, L.dtype_code(w_full), L.ACC_F64, r, L.ptr(uni),
               int(s_begin), int(s_count), a.data_ptr(), self.status.data_ptr(), ws, wsb, L.stream_handle())
        return a[:s_count]

    def permute_range(self, a_full, base, n_loc):
        """this rank's indices of permute_parallel (ancestry.py:139-174) over
        the full ancestry: (c_local, max steps, overflow)"""
        a_full = self._on_dev(torch.as_tensor(a_full).to(torch.int32))
        n = a_full.numel()
        c = torch.empty(max(n_loc, 1), dtype=torch.int32, device=self.dev)
        st = torch.zeros(1, dtype=torch.int32, device=self.dev)
        flag = torch.zeros(1, dtype=torch.int32, device=self.dev)
        ws, wsb = self._workspace(n)
        L.call("pfr_permute_range", a_full.data_ptr(), n, int(base), int(n_loc), c.data_ptr(), st.data_ptr(),
               flag.data_ptr(), ws, wsb, L.stream_handle())
        return c[:n_loc], st, flag

    def overflowed(self, flag) -> bool:
        return bool(L.read_status(flag) & L.ST_OVERFLOW)

    def permute(self, a_full):
        """the replicated full permute (fallback of permute_range)"""
        a_full = self._on_dev(torch.as_tensor(a_full).to(torch.int32))
        n = a_full.numel()
        c = torch.empty(n, dtype=torch.int32, device=self.dev)
        ws, wsb = self._workspace(n)
        L.call("pfr_permute", a_full.data_ptr(), n, L.I32, c.data_ptr(), None, self.status.data_ptr(), ws, wsb,
               L.stream_handle())
        return c


# ---------------------------------------------------------------------------
# the protocol


def shard_bounds(sizes):
    """Start index of every shard (rank order) and N."""
    offs = np.concatenate([[0], np.cumsum(np.asarray(sizes, dtype=np.int64))])
    return offs, int(offs[-1])


def _owner(idx: torch.Tensor, offs: np.ndarray) -> torch.Tensor:
    """rank owning each global index (shards are contiguous, in rank order)"""
    b = torch.as_tensor(offs[1:-1], dtype=torch.int64, device=idx.device)
    return torch.bucketize(idx.to(torch.int64), b, right=True)


def _route(rows: torch.Tensor, key_col: int, offs: np.ndarray, comm, width: int) -> torch.Tensor:
    """send each row to the rank owning rows[:, key_col]; returns the rows received"""
    if rows.shape[0]:
        dest = _owner(rows[:, key_col], offs)
        order = torch.argsort(dest, stable=True)
        rows = rows[order]
        counts = torch.bincount(dest, minlength=comm.world).cpu().tolist()
    else:
        counts = [0] * comm.world
    return comm.all_to_all(rows.contiguous(), counts, width).reshape(-1, width)


def _fold(values):
    """left fold in float64, the same association on every rank"""
    acc = 0.0
    out = []
    for v in values:
        out.append(acc)
        acc = acc + float(v)
    return out, acc


def _on_rank_stream(fn):
    """run a protocol entry point on the communicator's own stream, if it has
    one (virtual ranks), and hand the results back complete"""
    import functools

    @functools.wraps(fn)
    def wrapper(*args, comm, **kw):
        stream = getattr(comm, "stream", None)
        if stream is None:
            return fn(*args, comm=comm, **kw)
        stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(stream):
            out = fn(*args, comm=comm, **kw)
        stream.synchronize()
        return out

    return wrapper


@_on_rank_stream
def deliver_sharded(w_local, config, rng, *, comm, ops=None, rng_mode=None, uniforms=None,
                    return_max_steps: bool = False):
    """permute_parallel(resample_ancestors(w, config, rng).ancestors) for the
    global weight vector w = concat(shards in rank order); returns this rank's
    slice c[base:base+n_local] (global parent indices, int32).

    systematic / stratified: weight-sharded (see module docstring);
    metropolis / rejection: chains / slots partitioned over the all-gathered
    weights; multinomial: replicated over the all-gathered weights."""
    ops = ops or CudaShardOps()
    ops.reset()
    alg = config.algorithm
    if alg in ("systematic", "stratified"):
        return _deliver_offspring_sharded(w_local, alg == "stratified", rng, comm, ops, rng_mode, uniforms,
                                          return_max_steps)
    w_local = torch.as_tensor(w_local)
    # one exchange before the data moves: shard sizes and this shard's
    # validation bits (check_weights, diagnostics.py:38-51), so every rank
    # raises together and no rank waits in a collective another has left
    ops.check_local(w_local)
    rows = comm.all_gather_scalars(int(w_local.numel()) | (int(ops.status_bits()) << 40), torch.int64)
    sizes = [int(r) & ((1 << 40) - 1) for r in rows]
    bits = 0
    for r in rows:
        bits |= int(r) >> 40
    L.raise_weight_errors(bits, "w", True)
    offs, n = shard_bounds(sizes)
    base, n_loc = int(offs[comm.rank]), sizes[comm.rank]
    w_full = comm.all_gather_var(w_local)
    if alg == "metropolis":
        a_loc = metropolis_sharded(w_local, config, rng, comm=comm, ops=ops, rng_mode=rng_mode, _w_full=w_full,
                                   _sizes=sizes)
    elif alg in ("rejection", "rejection-capped"):
        # slots partitioned like Metropolis' chains
        a_loc = ops.rejection_range(w_full, config, rng, rng_mode, base, n_loc)
    elif alg == "multinomial":
        a_loc = ops.multinomial_range(w_full, rng, rng_mode, base, n_loc, uniforms)
    else:
        raise ValueError(f"unknown algorithm {alg!r}")
    # the in-place ancestry of this rank's indices only (pfr_permute_range)
    a_full = comm.all_gather_var(a_loc)
    c, steps, flag = ops.permute_range(a_full, base, n_loc)
    over = 0
    for f in comm.all_gather_scalars(int(ops.overflowed(flag)), torch.int64):
        over |= int(f)
    if over:  # a chain beyond the walk bound somewhere: the replicated permute
        c = ops.permute(a_full)[base: base + n_loc]
        steps = None
    ops.check()
    if not return_max_steps:
        return c
    if steps is None:
        return c, None
    return c, int(max(comm.all_gather_scalars(int(L.read_status(steps)), torch.int64)))


@_on_rank_stream
def metropolis_sharded(w_local, config_or_b, rng, *, comm, ops=None, rng_mode=None, _w_full=None, _sizes=None):
    """metropolis_ancestors (resamplers.py:204-234) with the N chains split over
    the ranks: returns this rank's slice of the ancestry (global indices)."""
    from .resamplers import ResamplerConfig, resolve_metropolis_steps

    ops = ops or CudaShardOps()
    sizes = _sizes or [int(s) for s in comm.all_gather_scalars(int(w_local.numel()), torch.int64)]
    offs, n = shard_bounds(sizes)
    w_full = _w_full if _w_full is not None else comm.all_gather_var(torch.as_tensor(w_local))
    if isinstance(config_or_b, ResamplerConfig):
        b = resolve_metropolis_steps(w_full, config_or_b)
    else:
        b = int(config_or_b)
    return ops.metropolis_range(w_full, b, rng, rng_mode, int(offs[comm.rank]), sizes[comm.rank])


# how often each systematic/stratified protocol ran (diagnostics; tests)
protocol_counts = {"v2": 0, "general": 0}  # "v2": the halo protocol (v3 kernels)
_count_lock = threading.Lock()


def _count(path):
    with _count_lock:
        protocol_counts[path] += 1


def halo_width(n: int) -> int:
    """slots kept on each side of a shard boundary (protocol v2): the drift
    between slot and parent is ~sqrt(N) for i.i.d. weights and a
    loser chain moves by it every step (p99 ~10 steps, tails ~30), so 32
    sqrt(N) keeps nearly every chain inside; PFR_SHARD_HALO overrides"""
    env = os.environ.get("PFR_SHARD_HALO")
    if env:
        return max(int(env), 0)
    return max(4096, 32 * math.isqrt(max(n, 1)))


def _deliver_offspring_sharded(w_local, stratified, rng, comm, ops, rng_mode, uniforms, return_max_steps):
    """Protocol v3: the shard's local work through the single-GPU kernels
    (K1, K2w, K3w of pfr_deliver.cu), two host synchronisations in all (the
    shard sizes with the validation bits after K1, the status bits at the
    end); the shard END values (all-gather) and the boundary bands (to the
    two neighbours) move device to device."""
    rank, world = comm.rank, comm.world
    w_local = torch.as_tensor(w_local)
    n_loc = int(w_local.numel())
    if n_loc < 1:
        raise ValueError("every rank needs a non-empty weight shard")
    # 1. K1 over the shard: hierarchy, validation bits, END value (device)
    end = ops.local_end(w_local)
    rows = comm.all_gather_scalars(n_loc | (int(ops.status_bits()) << 40), torch.int64)
    sizes = [int(r) & ((1 << 40) - 1) for r in rows]
    bits = 0
    for r in rows:
        bits |= int(r) >> 40
    L.raise_weight_errors(bits, "w", True)
    offs, n = shard_bounds(sizes)
    base = int(offs[rank])
    halo = halo_width(n)
    slot_lo = ((base - halo) // 4) * 4  # 16-byte aligned window start
    slot_hi = base + n_loc + halo
    shift = (base - halo) - slot_lo
    # 2. END values device to device; weight before the shard and W_N as left
    #    folds in rank order (the same IEEE additions on every rank)
    pt = ops.prefix_total(comm.all_gather_fixed(end), rank)
    # 3. K2w: O in global slot numbers and the slot words of this shard's window
    offset = 0.0 if stratified else ops.systematic_offset(rng, rng_mode)
    ext = torch.empty(slot_hi - slot_lo, dtype=torch.int32, device=end.device)
    ops.shard_produce(w_local, base, n, pt, rank == 0, rank == world - 1, stratified, offset, uniforms, rng, rng_mode,
                      ext, slot_lo, slot_hi)
    # 4. boundary bands to and from the two neighbours (point to point)
    view = ext[shift:]
    ops.merge(view, n_loc, halo, *comm.neighbor_exchange(*ops.bands(view, n_loc, halo)))
    # 5. K3w: the in-place ancestry of this shard's indices
    c, steps = ops.shard_resolve_fast(ext, slot_lo, slot_hi, base, n_loc, w_local.dtype)
    rows = comm.all_gather_scalars(int(ops.status_bits()) | (int(L.read_status(steps)) << 32), torch.int64)
    bits = 0
    for r in rows:
        bits |= int(r) & 0xFFFFFFFF
    if bits & L.ST_OVERFLOW:  # a drift or chain beyond the halo somewhere: the general protocol
        ops.reset()
        _count("general")
        return _deliver_offspring_general(w_local, stratified, rng, comm, ops, rng_mode, uniforms, return_max_steps)
    _count("v2")
    ops.check()
    if return_max_steps:
        return c, max(int(r) >> 32 for r in rows)
    return c


def _deliver_offspring_general(w_local, stratified, rng, comm, ops, rng_mode, uniforms, return_max_steps):
    """the general protocol (variable slot-word all-to-all, walker rounds): the
    fallback when a drift or a loser chain reaches beyond the halo"""
    rank, world = comm.rank, comm.world
    w_local = torch.as_tensor(w_local)
    sizes = [int(s) for s in comm.all_gather_scalars(int(w_local.numel()), torch.int64)]
    offs, n = shard_bounds(sizes)
    base, n_loc = int(offs[rank]), sizes[rank]
    if n_loc < 1:
        raise ValueError("every rank needs a non-empty weight shard")

    # 1. local scan, all-gather of shard totals -> prefix before this shard, W_N
    W_loc, t_loc = ops.local_scan(w_local)
    totals = comm.all_gather_scalars(float(t_loc), torch.float64)
    # validation bits travel with the totals so every rank raises together
    bits = 0
    for b in comm.all_gather_scalars(ops.status_bits(), torch.int64):
        bits |= int(b)
    L.raise_weight_errors(bits & ~L.ST_POSITIVE, "w", False)
    prefixes, total = _fold(totals)
    if not total > 0:
        raise ValueError("w must contain at least one strictly positive weight")

    # 2. offspring of this rank's parents in global slot numbers
    offset = 0.0 if stratified else ops.systematic_offset(rng, rng_mode)
    O = ops.offspring(W_loc, w_local.dtype, prefixes[rank], total, n, rank == world - 1, stratified, offset,
                      uniforms, rng, rng_mode)
    ends = [int(e) for e in comm.all_gather_scalars(int(O[-1].item()), torch.int64)]
    o_begin = ends[rank - 1] if rank else 0
    o_end = ends[rank]

    # 3. slot words of this rank's slot window -> the owners of those indices
    words, has = ops.words(O, base, o_begin)
    send = [max(0, min(o_end, int(offs[r + 1])) - max(o_begin, int(offs[r]))) for r in range(world)]
    words_here = comm.all_to_all(words, send, 1).reshape(-1)
    if words_here.numel() != n_loc:
        raise RuntimeError(f"sharded delivery: received {words_here.numel()} slot words for {n_loc} indices")

    # 4. local resolution, then walkers across shard boundaries
    c, pend, steps = ops.resolve(words_here, has, base)
    while True:
        counts = comm.all_gather_scalars(int(pend.shape[0]), torch.int64)
        if sum(counts) == 0:
            break
        arrived = _route(pend, 1, offs, comm, 3)
        done, fwd, st = ops.advance(arrived, words_here, base, n_loc)
        steps = max(steps, st)
        back = _route(done, 0, offs, comm, 2)
        ops.scatter(back, base, c)
        pend = fwd
    ops.check()
    if return_max_steps:
        return c, int(max(comm.all_gather_scalars(int(steps), torch.int64)))
    return c
