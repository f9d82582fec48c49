"""Ancestry conversions and the in-place permutation on the GPU.

Mirrors pfresample.ancestry (ancestry.py:69-174).  ``permute_parallel``
returns exactly the reference's vector for every input (the claim-and-chase
outcome is schedule independent, see csrc/pfr_ancestry.cu), computed by
atomic-min claims and bounded chain walks with a pointer-jumping fallback.
``permute_cumulative`` goes straight from a cumulative offspring vector to
the permuted ancestry without materialising the sorted ancestry.
"""

from __future__ import annotations

import torch

from . import _lib as L

__all__ = [
    "ancestors_to_offspring",
    "cumulative_offspring_to_ancestors",
    "cumulative_to_offspring",
    "offspring_to_cumulative",
    "prepermute",
    "permute_parallel",
    "permute_cumulative",
    "permute_serial",
    "satisfies_inplace_predicate",
    "copy_particles",
]


def _idx(a, name):
    return L.as_index(a, name)


def _finish_index(st, n):
    if L.config.check:
        L.raise_index_errors(L.read_status(st), n)


def cumulative_offspring_to_ancestors(O, *, index_dtype=None) -> torch.Tensor:
    """Parent i fills slots [O[i-1], O[i]) (ancestry.py:69-76); merge-path expand."""
    O = _idx(O, "cumulative offspring vector")
    n = O.numel()
    a = torch.empty(n, dtype=torch.int32, device=O.device)
    st = L.new_status()
    ws, wsb = L.workspace(n)
    L.call("pfr_cumulative_to_ancestors", O.data_ptr(), n, L.dtype_code(O), a.data_ptr(), st.data_ptr(), ws, wsb,
           L.stream_handle())
    _finish_index(st, n)
    return L.to_index_dtype(a, index_dtype)


def ancestors_to_offspring(a, *, index_dtype=None) -> torch.Tensor:
    """o[j] = #{i : a[i] = j} (ancestry.py:79-82)."""
    a = _idx(a, "ancestry vector")
    n = a.numel()
    o = torch.empty(n, dtype=torch.int32, device=a.device)
    st = L.new_status()
    L.call("pfr_ancestors_to_offspring", a.data_ptr(), n, L.dtype_code(a), o.data_ptr(), st.data_ptr(),
           L.stream_handle())
    _finish_index(st, n)
    return L.to_index_dtype(o, index_dtype)


def offspring_to_cumulative(o, *, index_dtype=None) -> torch.Tensor:
    """Inclusive integer scan with the reference's checks (ancestry.py:57-66, 85-88)."""
    o = _idx(o, "offspring vector")
    n = o.numel()
    out = torch.empty(n, dtype=torch.int64, device=o.device)
    st = L.new_status()
    ws, wsb = L.workspace(n)
    L.call("pfr_scan", o.data_ptr(), out.data_ptr(), n, L.dtype_code(o), L.I64, L.SCAN_EXPECT_N, 0, None,
           st.data_ptr(), ws, wsb, L.stream_handle())
    if L.config.check:
        bits = L.read_status(st)
        if bits & L.ST_NEGCOUNT:
            raise ValueError("offspring counts must be non-negative")
        if bits & L.ST_BADSUM:
            raise ValueError(f"offspring counts must sum to N={n}, got {int(out[-1])}")
    return L.to_index_dtype(out, index_dtype)


def cumulative_to_offspring(O, *, index_dtype=None) -> torch.Tensor:
    """Adjacent difference with the reference's checks (ancestry.py:44-54, 91-94)."""
    O = _idx(O, "cumulative offspring vector")
    n = O.numel()
    out = torch.empty(n, dtype=torch.int64, device=O.device)
    st = L.new_status()
    L.call("pfr_adjacent_difference", O.data_ptr(), out.data_ptr(), n, L.dtype_code(O), L.I64, st.data_ptr(),
           L.stream_handle())
    _finish_index(st, n)
    return L.to_index_dtype(out, index_dtype)


def satisfies_inplace_predicate(c) -> bool:
    """o[i] > 0 implies c[i] == i (ancestry.py:97-101)."""
    c = _idx(c, "ancestry vector")
    n = c.numel()
    res = torch.empty(1, dtype=torch.int32, device=c.device)
    st = L.new_status()
    ws, wsb = L.workspace(n)
    L.call("pfr_check_predicate", c.data_ptr(), n, L.dtype_code(c), res.data_ptr(), st.data_ptr(), ws, wsb,
           L.stream_handle())
    _finish_index(st, n)
    return bool(res.item())


def prepermute(a, *, index_dtype=None) -> torch.Tensor:
    """d[v] = lowest slot whose parent is v, sentinel N (ancestry.py:125-136)."""
    a = _idx(a, "ancestry vector")
    n = a.numel()
    d = torch.empty(n, dtype=torch.int32, device=a.device)
    st = L.new_status()
    L.call("pfr_prepermute", a.data_ptr(), n, L.dtype_code(a), d.data_ptr(), st.data_ptr(), L.stream_handle())
    _finish_index(st, n)
    return L.to_index_dtype(d, index_dtype)


def permute_parallel(a, return_max_steps: bool = False, *, index_dtype=None):
    """Claim-and-chase permutation satisfying o[i] > 0 => c[i] = i
    (ancestry.py:139-174); identical output to the reference."""
    a = _idx(a, "ancestry vector")
    n = a.numel()
    c = torch.empty(n, dtype=torch.int32, device=a.device)
    steps = torch.zeros(1, dtype=torch.int32, device=a.device) if return_max_steps else None
    st = L.new_status()
    ws, wsb = L.workspace(n)
    L.call("pfr_permute", a.data_ptr(), n, L.dtype_code(a), c.data_ptr(), L.ptr(steps), st.data_ptr(), ws, wsb,
           L.stream_handle())
    _finish_index(st, n)
    c = L.to_index_dtype(c, index_dtype)
    if return_max_steps:
        return c, int(steps.item())
    return c


def permute_cumulative(O, return_max_steps: bool = False, *, index_dtype=None):
    """permute_parallel(cumulative_offspring_to_ancestors(O)) without the
    intermediate sorted ancestry."""
    O = _idx(O, "cumulative offspring vector").to(torch.int32)
    n = O.numel()
    c = torch.empty(n, dtype=torch.int32, device=O.device)
    steps = torch.zeros(1, dtype=torch.int32, device=O.device) if return_max_steps else None
    st = L.new_status()
    ws, wsb = L.workspace(n)
    L.call("pfr_permute_cumulative", O.data_ptr(), n, c.data_ptr(), L.ptr(steps), st.data_ptr(), ws, wsb,
           L.stream_handle())
    c = L.to_index_dtype(c, index_dtype)
    if return_max_steps:
        return c, int(steps.item())
    return c


def permute_serial(a, *, index_dtype=None) -> torch.Tensor:
    """Serial pairwise-swap permutation (ancestry.py:104-122, PAPER Code 11)
    satisfying the in-place predicate; run by one device thread (the
    algorithm is inherently sequential -- permute_parallel is the
    production permutation; the two may differ element-wise)."""
    a = _idx(a, "ancestry vector")
    n = a.numel()
    c = torch.empty(n, dtype=torch.int32, device=a.device)
    st = L.new_status()
    L.call("pfr_permute_serial", a.data_ptr(), n, L.dtype_code(a), c.data_ptr(), st.data_ptr(), L.stream_handle())
    _finish_index(st, n)
    return L.to_index_dtype(c, index_dtype)


def copy_particles(x: torch.Tensor, c) -> torch.Tensor:
    """In-place x[i] = x[c[i]] where c[i] != i (pf.py:86-97); x is float64
    with shape (N,) or (N, width); c must satisfy the in-place predicate."""
    c = _idx(c, "ancestry vector").to(torch.int32)
    if x.dtype != torch.float64 or not x.is_contiguous() or x.device != c.device:
        raise ValueError("x must be a contiguous float64 tensor on the ancestry's device")
    n = c.numel()
    if x.shape[0] != n:
        raise ValueError(f"x has {x.shape[0]} particles but the ancestry vector has {n} entries")
    if L.config.check and n and (int(c.min()) < 0 or int(c.max()) >= n):
        raise ValueError(f"ancestry entries must lie in [0, {n})")  # an out-of-range c would read outside x
    width = x.numel() // n if n else 1
    L.call("pfr_copy_particles", x.data_ptr(), n, width, c.data_ptr(), L.stream_handle())
    return x
