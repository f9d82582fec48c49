"""CPU stand-in for paper_1301_4019_b200.sharded.CudaShardOps -- TEST
INFRASTRUCTURE ONLY.

Implements the per-rank operations of the sharded protocol with NumPy and the
oracle (oracle/pfr_oracle.py), with exactly the semantics the CUDA kernels of
csrc/pfr_shard.cu document, so that the host protocol (collectives, routing,
walker rounds) can be exercised on CPU with gloo or ThreadComm.  The product
path never imports this module.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import pfr_oracle as orc

FIRST = 0x80000000
MASK = 0x7FFFFFFF


def _np(t, dtype=None):
    a = t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
    return a if dtype is None else a.astype(dtype)


def _word(v):
    return int(v) & 0xFFFFFFFF


class NumpyShardOps:
    def __init__(self):
        self.bits = 0

    def status_bits(self):
        return self.bits

    def reset(self):
        self.bits = 0

    def check(self):
        pass

    def check_local(self, w_local):
        from paper_1301_4019_b200 import _lib as L

        w = _np(w_local)
        if not np.all(np.isfinite(w)):
            self.bits |= L.ST_NONFINITE
        if np.any(w < 0):
            self.bits |= L.ST_NEGATIVE
        if np.any(w > 0):
            self.bits |= L.ST_POSITIVE

    def local_scan(self, w):
        w = _np(w)
        if not np.all(np.isfinite(w)):
            self.bits |= 1
        if np.any(w < 0):
            self.bits |= 2
        W = np.cumsum(w.astype(np.float64))
        return torch.from_numpy(W), float(W[-1])

    def systematic_offset(self, rng, mode):
        assert mode == "numpy", "the CPU stand-in replays the reference stream only"
        return orc.systematic_offset(rng.seed, rng.ids)

    def offspring(self, W, wdtype, prefix, total, n_global, last, stratified, offset, uniforms, rng, mode):
        W = prefix + _np(W, np.float64)
        r = (W * float(n_global)) / total
        k = np.clip(np.floor(r).astype(np.int64) + 1, 1, n_global)
        if stratified:
            u_all = (np.asarray(uniforms, dtype=np.float64) if uniforms is not None
                     else orc.stratified_uniforms(rng.seed, rng.ids, n_global))
            u = u_all[k - 1]
        else:
            u = np.full(W.size, offset, dtype=np.float64)
        if wdtype == torch.float32:
            u = u.astype(np.float32).astype(np.float64)
        O = np.clip(np.floor(r + u).astype(np.int64), 0, n_global)
        if last:
            O[-1] = n_global
        return torch.from_numpy(O.astype(np.int32))

    def words(self, O, base, o_begin):
        O = _np(O, np.int64)
        prev = np.concatenate([[o_begin], O[:-1]])
        o = O - prev
        if np.any(o < 0):
            self.bits |= 1 << 7
        o = np.maximum(o, 0)
        parents = np.repeat(base + np.arange(O.size, dtype=np.int64), o)
        words = parents.copy()
        words[(prev[o > 0] - o_begin)] |= FIRST
        return torch.from_numpy(words.astype(np.uint32).view(np.int32)), torch.from_numpy((o > 0).astype(np.uint8))

    def _walk(self, wd, words, base, n, steps):
        while wd & FIRST:
            y = wd & MASK
            steps += 1
            if y < base or y >= base + n:
                return None, y, steps
            wd = _word(words[y - base])
        return wd & MASK, None, steps

    def resolve(self, words, has, base):
        words = _np(words)
        has = _np(has)
        n = has.size
        c = np.empty(n, dtype=np.int32)
        pend, longest = [], 0
        for i in range(n):
            if has[i]:
                c[i] = base + i
                continue
            v, z, st = self._walk(_word(words[i]), words, base, n, 0)
            if v is None:
                pend.append((base + i, z, st))
            else:
                c[i] = v
                longest = max(longest, st)
        return (torch.from_numpy(c), torch.tensor(pend, dtype=torch.int32).reshape(-1, 3), longest)

    def advance(self, walkers, words, base, n_loc):
        words = _np(words)
        done, fwd, longest = [], [], 0
        for h, z0, st in _np(walkers).reshape(-1, 3).tolist():
            assert base <= z0 < base + n_loc
            v, z, st = self._walk(_word(words[z0 - base]), words, base, n_loc, st)
            if v is None:
                fwd.append((h, z, st))
            else:
                done.append((h, v))
                longest = max(longest, st)
        return (torch.tensor(done, dtype=torch.int32).reshape(-1, 2), torch.tensor(fwd, dtype=torch.int32).reshape(-1, 3),
                longest)

    def scatter(self, done, base, c):
        for h, v in _np(done).reshape(-1, 2).tolist():
            c[h - base] = v

    # ---- protocol v3 (pfr_shard_local_end / _produce / _resolve_fast), in NumPy
    def local_end(self, w):
        self.check_local(w)  # K1 reports check_weights' flags, the positive one included
        W, _ = self.local_scan(w)
        return W[-1:].clone()

    def shard_produce(self, w, base, n_global, pt, first, last, stratified, offset, uniforms, rng, mode, ext, slot_lo,
                      slot_hi):
        from paper_1301_4019_b200 import _lib as L

        W, _ = self.local_scan(w)
        wdtype = torch.as_tensor(w).dtype
        O, ob = self.offspring_dev(W, wdtype, pt, n_global, last, first, stratified, offset, uniforms, rng, mode)
        O = _np(O, np.int64)
        prev = np.concatenate([[int(_np(ob)[0])], O[:-1]])
        o = O - prev
        if np.any(o < 0):
            self.bits |= L.ST_OVERFLOW
        e = ext.numpy().view(np.uint32)
        e[:] = self.SENT
        self._has = (o > 0).astype(np.uint8)
        for i in np.flatnonzero(o > 0).tolist():
            for sl in range(int(prev[i]), int(O[i])):
                if slot_lo <= sl < slot_hi:
                    e[sl - slot_lo] = (base + i) | (FIRST if sl == prev[i] else 0)
                else:
                    self.bits |= L.ST_OVERFLOW

    def shard_resolve_fast(self, ext, slot_lo, slot_hi, base, n_loc, wdtype):
        halo = base - slot_lo  # resolve_ext's extended array starts at base - halo
        c, st = self.resolve_ext(ext, n_loc, halo, torch.from_numpy(self._has), base)
        return c, st

    # ---- protocol v2 (csrc/pfr_shard.cu: k_shard_offspring_dev, k_shard_ext_words,
    # k_shard_merge, k_shard_resolve_ext), in NumPy
    SENT = 0xFFFFFFFF

    def local_scan_dev(self, w):
        W, t = self.local_scan(w)
        return W, W[-1:].clone()

    def prefix_total(self, totals, rank):
        totals = _np(totals, np.float64)
        acc, prefix = 0.0, 0.0
        for r, v in enumerate(totals.tolist()):
            if r == rank:
                prefix = acc
            acc = acc + v
        return torch.tensor([prefix, acc], dtype=torch.float64)

    def offspring_dev(self, W, wdtype, pt, n_global, last, first, stratified, offset, uniforms, rng, mode):
        prefix, total = _np(pt, np.float64).tolist()
        O = self.offspring(W, wdtype, prefix, total, n_global, last, stratified, offset, uniforms, rng, mode)
        if first:
            ob = 0
        else:  # the formula at W = prefix (the previous shard's last element)
            ob = int(self.offspring(torch.zeros(1, dtype=torch.float64), wdtype, prefix, total, n_global, False,
                                    stratified, offset, uniforms, rng, mode)[0])
        return O, torch.tensor([ob], dtype=torch.int32)

    def ext_words(self, O, base, o_before, halo):
        from paper_1301_4019_b200 import _lib as L

        O = _np(O, np.int64)
        n = O.size
        ext = np.full(n + 2 * halo, self.SENT, dtype=np.uint64)
        prev = np.concatenate([[int(_np(o_before)[0])], O[:-1]])
        o = O - prev
        if np.any(o < 0):
            self.bits |= L.ST_NOTMONOTONE
        has = (o > 0).astype(np.uint8)
        lo_slot = base - halo
        for i in np.flatnonzero(o > 0).tolist():
            for sl in range(int(prev[i]), int(O[i])):
                pos = sl - lo_slot
                if 0 <= pos < ext.size:
                    ext[pos] = (base + i) | (FIRST if sl == prev[i] else 0)
                else:
                    self.bits |= L.ST_OVERFLOW
        return torch.from_numpy(ext.astype(np.uint32).view(np.int32)), torch.from_numpy(has)

    @staticmethod
    def bands(ext, n_loc, halo):
        return ext[: 2 * halo], ext[n_loc: n_loc + 2 * halo]

    def merge(self, ext, n_loc, halo, from_left, from_right):
        e = ext.numpy().view(np.uint32)
        if from_left is not None:
            src = _np(from_left).view(np.uint32)
            m = (src != self.SENT) & (e[: 2 * halo] == self.SENT)
            e[: 2 * halo][m] = src[m]
        if from_right is not None:
            src = _np(from_right).view(np.uint32)
            m = (src != self.SENT) & (e[n_loc: n_loc + 2 * halo] == self.SENT)
            e[n_loc: n_loc + 2 * halo][m] = src[m]

    def resolve_ext(self, ext, n_loc, halo, has, base):
        from paper_1301_4019_b200 import _lib as L

        e = ext.numpy().view(np.uint32)
        has = _np(has)
        c = np.empty(n_loc, dtype=np.int32)
        lo_slot, longest = base - halo, 0
        for i in range(n_loc):
            if has[i]:
                c[i] = base + i
                continue
            wd = int(e[halo + i])
            if wd == self.SENT:
                self.bits |= L.ST_OVERFLOW
                continue
            st, ok = 0, True
            while wd & FIRST:
                pos = (wd & MASK) - lo_slot
                st += 1
                if st > 4096 or pos < 0 or pos >= e.size or int(e[pos]) == self.SENT:
                    ok = False
                    break
                wd = int(e[pos])
            if not ok:
                self.bits |= L.ST_OVERFLOW
                continue
            c[i] = wd & MASK
            longest = max(longest, st)
        return torch.from_numpy(c), torch.tensor([longest], dtype=torch.int32)

    def metropolis_range(self, w_full, b, rng, mode, c_begin, c_count):
        a = orc.metropolis_stream(_np(w_full), b, rng.seed, rng.ids)
        return torch.from_numpy(a[c_begin: c_begin + c_count].astype(np.int32))

    def rejection_range(self, w_full, config, rng, mode, s_begin, s_count):
        # the reference's rejection loop is round-synchronous over the whole
        # pending set (not slot-separable): the CPU stand-in slices the full run
        w = _np(w_full)
        sup = config.sup_w if config.sup_w is not None else float(w.max())
        a = orc.rejection_stream(w, sup, rng.seed, rng.ids)[0]
        return torch.from_numpy(a[s_begin: s_begin + s_count].astype(np.int32))

    def multinomial_range(self, w_full, rng, mode, s_begin, s_count, uniforms=None):
        a = orc.multinomial_stream(_np(w_full), rng.seed, rng.ids)
        return torch.from_numpy(a[s_begin: s_begin + s_count].astype(np.int32))

    def permute_range(self, a_full, base, n_loc):
        """the backward walks of csrc/pfr_ancestry.cu's k_permute_range, in NumPy"""
        a = _np(a_full, np.int64)
        n = a.size
        d = orc.prepermute(a)
        c = np.empty(n_loc, dtype=np.int32)
        longest = 0
        for t in range(n_loc):
            x = base + t
            if d[x] < n:
                c[t] = x
                continue
            z, hops = x, 0
            while d[a[z]] == z:
                z = a[z]
                hops += 1
            c[t] = a[z]
            longest = max(longest, hops)
        return torch.from_numpy(c), torch.tensor([longest], dtype=torch.int32), torch.zeros(1, dtype=torch.int32)

    def overflowed(self, flag):
        return False

    def permute(self, a_full):
        return torch.from_numpy(orc.permute(_np(a_full)).astype(np.int32))
