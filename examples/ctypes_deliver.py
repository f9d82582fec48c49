"""The C ABI without torch: a systematic delivery through ctypes, with device
memory from cuda-python (cuda.bindings.runtime) -- what a non-Python host
(cgo / JNI / N-API) would do through its own FFI.  Prints the in-place
ancestry's check and exits non-zero on failure.

    python examples/ctypes_deliver.py [N]
"""
import ctypes
import os
import sys

import numpy as np
from cuda.bindings import runtime as rt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_1301_4019_b200", "libpfr.so"))


class PfrRng(ctypes.Structure):
    _fields_ = [("key0", ctypes.c_uint64), ("key1", ctypes.c_uint64), ("mode", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


P, I64, INT, DBL, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
lib.pfr_workspace_bytes.argtypes = [INT, I64, INT]
lib.pfr_workspace_bytes.restype = SZ
lib.pfr_deliver_offspring.argtypes = [P, I64, INT, INT, INT, DBL, P, ctypes.POINTER(PfrRng), P, P, P, P, P, SZ, P]
lib.pfr_deliver_offspring.restype = INT
lib.pfr_last_error.restype = ctypes.c_char_p
PFR_OP_ANY, PFR_F32, PFR_ACC_F64 = 10, 0, 0  # include/pfr.h enums


def check(err):
    err = err[0] if isinstance(err, tuple) else err
    if err != rt.cudaError_t.cudaSuccess:
        raise RuntimeError(f"CUDA error {err}")


def dmalloc(nbytes):
    err, ptr = rt.cudaMalloc(nbytes)
    check(err)
    return ptr


def main(n):
    w = np.exp(np.random.default_rng(1).normal(0, 1, n)).astype(np.float32)
    ws_bytes = lib.pfr_workspace_bytes(PFR_OP_ANY, n, PFR_F32)
    w_dev, c_dev, st_dev, ws_dev = dmalloc(4 * n), dmalloc(4 * n), dmalloc(4), dmalloc(ws_bytes)
    check(rt.cudaMemset(ws_dev, 0, ws_bytes))  # zero-filled once per workspace
    check(rt.cudaMemset(st_dev, 0, 4))
    check(rt.cudaMemcpy(w_dev, w.ctypes.data, 4 * n, rt.cudaMemcpyKind.cudaMemcpyHostToDevice))
    rng = PfrRng(0x1234, 0x5678, 0, 0)  # PFR_RNG_PHILOX; keys = derive_seed(seed, 0|1, *ids)
    rc = lib.pfr_deliver_offspring(w_dev, n, PFR_F32, PFR_ACC_F64, 0, 0.25, None, ctypes.byref(rng), c_dev, None,
                                   None, st_dev, ws_dev, ws_bytes, None)  # default stream
    if rc != 0:
        raise RuntimeError(lib.pfr_last_error().decode())
    check(rt.cudaDeviceSynchronize())
    c = np.empty(n, dtype=np.int32)
    status = np.zeros(1, dtype=np.uint32)
    check(rt.cudaMemcpy(c.ctypes.data, c_dev, 4 * n, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost))
    check(rt.cudaMemcpy(status.ctypes.data, st_dev, 4, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost))
    for p in (w_dev, c_dev, st_dev, ws_dev):
        check(rt.cudaFree(p))
    o = np.bincount(c, minlength=n)
    ok = bool(np.all(c[o > 0] == np.flatnonzero(o > 0)))  # o[i] > 0 => c[i] = i (ancestry.py:97-101)
    # systematic with offset u: o[i] within 1 of N w_i / W
    m = n * w.astype(np.float64) / w.astype(np.float64).sum()
    ok &= bool(np.abs(o - m).max() < 1.0 + 1e-6)
    print(f"N={n}: status bits {int(status[0]):#x}, in-place predicate and systematic bounds "
          f"{'hold' if ok else 'FAIL'}")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20))
