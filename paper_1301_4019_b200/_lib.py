"""ctypes binding of libpfr.so and the host-side plumbing shared by the API
modules: device tensors, the caller's CUDA stream, the per-device workspace,
the status word and the mapping of status bits onto the reference's
exceptions.

There is deliberately no CPU implementation behind this module: if the
library cannot be loaded or no CUDA device is present, every call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpfr.so")

# --- constants mirrored from include/pfr.h ----------------------------------
F32, F64, I32, I64 = 0, 1, 2, 3
ACC_F64, ACC_NATIVE, ACC_SERIAL = 0, 1, 2
SCAN_MONOTONE = 0x100
SCAN_EXPECT_N = 0x200
RNG_PHILOX, RNG_NUMPY, RNG_ARRAYS = 0, 1, 2

ST_NONFINITE = 1 << 0
ST_NEGATIVE = 1 << 1
ST_POSITIVE = 1 << 2
ST_RANGE = 1 << 3
ST_REPAIRED = 1 << 4
ST_OVERFLOW = 1 << 5
ST_NOPROGRESS = 1 << 6
ST_NOTMONOTONE = 1 << 7
ST_BADEND = 1 << 8
ST_NEGCOUNT = 1 << 9
ST_BADSUM = 1 << 10
ST_RATIO = 1 << 11
ST_NONTERMINATION = 1 << 12

E_OK, E_ARG, E_WORKSPACE, E_CUDA, E_UNSUPPORTED = 0, 1, 2, 3, 4

OP_SCAN, OP_OFFSPRING, OP_DELIVER, OP_PERMUTE, OP_MULTINOMIAL = 0, 1, 2, 3, 4
OP_METROPOLIS, OP_REJECTION, OP_EXPAND, OP_LOGWEIGHTS, OP_PREDICATE, OP_ANY = 5, 6, 7, 8, 9, 10


class PfrRng(ctypes.Structure):
    _fields_ = [("key0", ctypes.c_uint64), ("key1", ctypes.c_uint64), ("mode", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_INT = ctypes.c_int
_DBL = ctypes.c_double
_SZ = ctypes.c_size_t
_RNGP = ctypes.POINTER(PfrRng)

_SIGNATURES = {
    "pfr_abi_version": ([], _INT),
    "pfr_last_error": ([], ctypes.c_char_p),
    "pfr_workspace_bytes": ([_INT, _I64, _INT], _SZ),
    "pfr_launch_count": ([_INT], ctypes.c_uint64),
    "pfr_stream_uniform": ([_RNGP, ctypes.c_uint64, ctypes.c_uint32], _DBL),
    "pfr_scan": ([_P, _P, _I64, _INT, _INT, _INT, _INT, _P, _P, _P, _SZ, _P], _INT),
    "pfr_adjacent_difference": ([_P, _P, _I64, _INT, _INT, _P, _P], _INT),
    "pfr_lower_bound": ([_P, _I64, _INT, _P, _I64, _P, _P], _INT),
    "pfr_check_weights": ([_P, _I64, _INT, _P, _P], _INT),
    "pfr_logweights_to_weights": ([_P, _P, _I64, _INT, _P, _P, _SZ, _P], _INT),
    "pfr_cumulative_offspring": ([_P, _I64, _INT, _INT, _INT, _DBL, _P, _RNGP, _P, _P, _P, _SZ, _P], _INT),
    "pfr_deliver_offspring": ([_P, _I64, _INT, _INT, _INT, _DBL, _P, _RNGP, _P, _P, _P, _P, _P, _SZ, _P], _INT),
    "pfr_deliver_offspring_logw": ([_P, _I64, _INT, _INT, _INT, _DBL, _P, _RNGP, _P, _P, _P, _P, _P, _SZ, _P], _INT),
    "pfr_multinomial": ([_P, _I64, _INT, _INT, _RNGP, _P, _INT, _P, _P, _P, _SZ, _P], _INT),
    "pfr_metropolis": ([_P, _I64, _INT, _I64, _RNGP, _P, _P, _INT, _P, _P, _P, _SZ, _P], _INT),
    "pfr_rejection": ([_P, _I64, _INT, _DBL, _DBL, _RNGP, _I64, _P, _P, _P, _P, _P, _SZ, _P], _INT),
    "pfr_rejection_range": ([_P, _I64, _INT, _DBL, _DBL, _RNGP, _I64, _I64, _I64, _P, _P, _P, _P, _P, _SZ, _P], _INT),
    "pfr_cumulative_to_ancestors": ([_P, _I64, _INT, _P, _P, _P, _SZ, _P], _INT),
    "pfr_ancestors_to_offspring": ([_P, _I64, _INT, _P, _P, _P], _INT),
    "pfr_prepermute": ([_P, _I64, _INT, _P, _P, _P], _INT),
    "pfr_permute": ([_P, _I64, _INT, _P, _P, _P, _P, _SZ, _P], _INT),
    "pfr_permute_cumulative": ([_P, _I64, _P, _P, _P, _P, _SZ, _P], _INT),
    "pfr_check_predicate": ([_P, _I64, _INT, _P, _P, _P, _SZ, _P], _INT),
    "pfr_copy_particles": ([_P, _I64, _I64, _P, _P], _INT),
    "pfr_metropolis_range": ([_P, _I64, _INT, _I64, _RNGP, _I64, _I64, _P, _P, _P], _INT),
    "pfr_shard_merge_bands": ([_P, _I64, _I64, _P, _P, _P], _INT),
    "pfr_shard_local_end": ([_P, _I64, _INT, _P, _P, _P, _SZ, _P], _INT),
    "pfr_shard_produce": ([_P, _I64, _INT, _I64, _I64, _P, _INT, _INT, _INT, _DBL, _P, _RNGP, _P, _I64, _I64, _P, _P,
                           _SZ, _P], _INT),
    "pfr_shard_resolve_fast": ([_I64, _INT, _I64, _P, _I64, _I64, _P, _P, _P, _P, _SZ, _P], _INT),
    "pfr_multinomial_range": ([_P, _I64, _INT, _INT, _RNGP, _P, _I64, _I64, _P, _P, _P, _SZ, _P], _INT),
    "pfr_permute_range": ([_P, _I64, _I64, _I64, _P, _P, _P, _P, _SZ, _P], _INT),
    "pfr_shard_offspring": ([_P, _I64, _INT, _DBL, _DBL, _I64, _INT, _INT, _DBL, _P, _RNGP, _P, _P], _INT),
    "pfr_shard_words": ([_P, _I64, _I64, ctypes.c_int32, _P, _P, _P, _P], _INT),
    "pfr_shard_resolve": ([_P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P], _INT),
    "pfr_shard_advance": ([_P, _I64, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P], _INT),
    "pfr_shard_scatter": ([_P, _I64, _I64, _I64, _P, _P, _P], _INT),
    "pfr_batched_workspace_bytes": ([_I64, _I64], _SZ),
    "pfr_deliver_batched": ([_P, _I64, _I64, _INT, _P, _RNGP, _P, _P, _P, _P, _SZ, _P], _INT),
    "pfr_pf_workspace_bytes": ([_I64, _I64], _SZ),
    "pfr_pf_run": ([_P, _P, _I64, _I64, _I64, _DBL, _RNGP, _P, _P, _P, _P, _P, _P, _SZ, _P], _INT),
    "pfr_permute_serial": ([_P, _I64, _INT, _P, _P, _P], _INT),
    "pfr_stable_sum": ([_P, _I64, _INT, _P, _P, _SZ, _P], _INT),
    "pfr_weight_stats": ([_P, _I64, _INT, _P, _INT, _P, _P, _SZ, _P], _INT),
    "pfr_probe_gather": ([_P, _I64, _INT, _I64, _P, _P], _INT),
    "pfr_deliver_metropolis": ([_P, _I64, _INT, _I64, _RNGP, _P, _P, _P, _P, _SZ, _P], _INT),
    "pfr_deliver_rejection": ([_P, _I64, _INT, ctypes.c_double, _RNGP, _I64, _P, _P, _P, _P, _SZ, _P], _INT),
    "pfr_deliver_multinomial": ([_P, _I64, _INT, _INT, _RNGP, _P, _P, _P, _P, _SZ, _P], _INT),
}

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load libpfr.so (no CUDA device needed to load it)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(paper_1301_4019_b200/_build.py); there is no CPU fallback")
            lib = ctypes.CDLL(path)
            for name, (args, res) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def lib():
    if _lib is None:
        load_library()
    return _lib


def exported_symbols():
    return list(_SIGNATURES)


# --- configuration ---------------------------------------------------------


@dataclass
class Config:
    """Process-wide defaults (each call can override)."""

    rng_mode: str = "philox"   # "philox" (own Philox4x32-10) or "numpy" (replay numpy's stream)
    accum: str = "f64"         # "f64" (fp32 is storage only), "native" (dtype arithmetic, tree association)
                               # or "serial" (np.cumsum bit for bit: the reference's fold, parity mode)
    index_dtype: torch.dtype = torch.int64
    check: bool = True         # synchronise and raise the reference's exceptions


config = Config()


def rng_mode_code(mode: str | None) -> int:
    mode = config.rng_mode if mode is None else mode
    if mode == "philox":
        return RNG_PHILOX
    if mode == "numpy":
        return RNG_NUMPY
    raise ValueError(f"unknown rng_mode {mode!r}; choose 'philox' or 'numpy'")


def accum_code(accum: str | None) -> int:
    accum = config.accum if accum is None else accum
    if accum == "f64":
        return ACC_F64
    if accum == "native":
        return ACC_NATIVE
    if accum == "serial":
        return ACC_SERIAL
    raise ValueError(f"unknown accum {accum!r}; choose 'f64', 'native' or 'serial'")


# --- tensors ---------------------------------------------------------------


_cuda_ok = False
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_get_device = getattr(torch._C, "_cuda_getDevice", None)


def _require_cuda() -> None:
    global _cuda_ok
    if not _cuda_ok:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1301_4019_b200 needs a CUDA device (B200); no CPU fallback exists")
        torch.cuda.init()
        _cuda_ok = True


def device() -> torch.device:
    _require_cuda()
    return torch.device("cuda", _get_device() if _get_device is not None else torch.cuda.current_device())


def stream_handle() -> int:
    """cudaStream_t of torch's current stream on the current device (the
    public accessors cost ~10 us of Python per call; the enqueue path uses
    torch's raw accessor when present)."""
    _require_cuda()
    if _raw_stream is not None and _get_device is not None:
        return _raw_stream(_get_device())
    return torch.cuda.current_stream().cuda_stream


def as_weights(w, name: str = "w") -> torch.Tensor:
    """1-D contiguous float32/float64 device tensor (non-float input -> float64),
    mirroring _as_vector / check_weights' conversion rules (primitives.py:23-31)."""
    dev = device()
    if isinstance(w, torch.Tensor):
        t = w
    else:
        arr = np.asarray(w)
        if arr.dtype.kind not in "f":
            arr = arr.astype(np.float64)
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.dim() != 1 or t.numel() < 1:
        raise ValueError(f"{name} must be a one-dimensional vector with at least one element")
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    t = t.to(dev, non_blocking=True)
    if not t.is_contiguous() or t.data_ptr() % 16:
        t = t.contiguous().clone()
    return t


def as_index(a, name: str = "ancestry vector") -> torch.Tensor:
    """1-D contiguous int32/int64 device tensor; integral floats accepted like
    _check_ancestry (ancestry.py:28-41)."""
    dev = device()
    if isinstance(a, torch.Tensor):
        t = a
    else:
        arr = np.asarray(a)
        if arr.dtype.kind == "f":
            if not np.all(arr == np.floor(arr)):
                raise ValueError(f"{name} must contain integers")
            arr = arr.astype(np.int64)
        elif arr.dtype.kind not in "iu":
            raise ValueError(f"{name} must contain integers")
        t = torch.from_numpy(np.ascontiguousarray(arr.astype(np.int64, copy=False)))
    if t.dim() != 1 or t.numel() < 1:
        raise ValueError(f"{name} must be one-dimensional and non-empty")
    if t.dtype.is_floating_point:
        if not bool(torch.all(t == torch.floor(t))):
            raise ValueError(f"{name} must contain integers")
        t = t.to(torch.int64)
    if t.dtype not in (torch.int32, torch.int64):
        t = t.to(torch.int64)
    t = t.to(dev, non_blocking=True)
    if not t.is_contiguous() or t.data_ptr() % 16:
        t = t.contiguous().clone()
    return t


def dtype_code(t: torch.Tensor) -> int:
    return {torch.float32: F32, torch.float64: F64, torch.int32: I32, torch.int64: I64}[t.dtype]


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


# --- workspace + status (per device and stream, grow-only) ------------------
# Calls on different streams may run concurrently (independent filters on
# their own streams), so each (device, stream) owns its workspace and its
# status words; calls on one stream are ordered by the stream.

_ws = {}
_status = {}
_ws_lock = threading.Lock()


def workspace(n: int) -> tuple[int, int]:
    dev = device()
    key = (dev.index, stream_handle())
    need = int(lib().pfr_workspace_bytes(OP_ANY, int(n), 0))
    cur = _ws.get(key)
    if cur is None or cur.numel() < need:
        # zero-filled once: the fused delivery keeps its counters in it (pfr.h)
        cur = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=dev)
        with _ws_lock:
            _ws[key] = cur
    return cur.data_ptr(), cur.numel()


_RING = 256  # status words per device, zeroed together


class _StatusRing:
    """A ring of device status words zeroed in bulk: each call takes a fresh
    zero word, so no per-call fill kernel sits on the stream; the ring is
    re-zeroed (one fill, ordered after every earlier user on the stream) when
    it wraps."""

    def __init__(self, dev):
        self.words = torch.zeros(_RING, dtype=torch.int32, device=dev)
        self.next = 0
        self.last = self.words[0:1]

    def take(self) -> torch.Tensor:
        if self.next == _RING:
            self.words.zero_()
            self.next = 0
        self.last = self.words[self.next: self.next + 1]
        self.next += 1
        return self.last


_rings = threading.local()


def _ring() -> _StatusRing:
    dev = device()
    rings = getattr(_rings, "by_dev", None)
    if rings is None:
        rings = _rings.by_dev = {}
    key = (dev.index, stream_handle())
    r = rings.get(key)
    if r is None:
        r = rings[key] = _StatusRing(dev)
    return r


def status_word() -> torch.Tensor:
    """The status word of the most recent call on this thread and device."""
    return _ring().last


def new_status() -> torch.Tensor:
    return _ring().take()


def status_all() -> int:
    """OR of every status word this thread handed out on the current device
    (all streams) since each ring last wrapped."""
    dev = device()
    _ring()
    acc = 0
    for (d, _), r in getattr(_rings, "by_dev", {}).items():
        if d == dev.index:
            acc |= int(np.bitwise_or.reduce(r.words[: max(r.next, 1)].cpu().numpy()))
    return acc & 0xFFFFFFFF


def read_status(st: torch.Tensor) -> int:
    return int(st.item()) & 0xFFFFFFFF


def call(name: str, *args) -> None:
    rc = getattr(lib(), name)(*args)
    if rc != E_OK:
        msg = lib().pfr_last_error().decode(errors="replace")
        if rc == E_ARG:
            raise ValueError(msg)
        if rc == E_UNSUPPORTED:
            raise NotImplementedError(msg)
        raise RuntimeError(f"{name} failed ({rc}): {msg}")


# --- status -> reference exceptions ------------------------------------------


def raise_weight_errors(bits: int, name: str = "w", require_positive_total: bool = True) -> None:
    """check_weights messages (diagnostics.py:38-51)."""
    if bits & ST_NONFINITE:
        raise ValueError(f"{name} must be finite (no NaN or infinity)")
    if bits & ST_NEGATIVE:
        raise ValueError(f"{name} must be non-negative")
    if require_positive_total and not bits & ST_POSITIVE:
        raise ValueError(f"{name} must contain at least one strictly positive weight")


def raise_index_errors(bits: int, n: int) -> None:
    if bits & ST_RANGE:
        raise ValueError(f"ancestry entries must lie in [0, {n})")
    if bits & (ST_NOTMONOTONE | ST_NEGCOUNT) and not bits & ST_BADSUM:
        raise ValueError("cumulative offspring vector must be non-negative and non-decreasing")
    if bits & ST_BADEND:
        raise ValueError(f"cumulative offspring vector must end at N={n}")


def to_index_dtype(t: torch.Tensor, index_dtype=None) -> torch.Tensor:
    want = config.index_dtype if index_dtype is None else index_dtype
    return t if t.dtype == want else t.to(want)
