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

    def check(self):
        pass

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

    def full_ancestors(self, w_full, config, rng, mode):
        w = _np(w_full)
        if config.algorithm == "multinomial":
            return torch.from_numpy(orc.multinomial_stream(w, rng.seed, rng.ids).astype(np.int32))
        raise NotImplementedError(config.algorithm)

    def permute(self, a_full):
        return torch.from_numpy(orc.permute(_np(a_full)).astype(np.int32))
