"""CPU checks of the C-ABI library: it loads, exports every symbol pfr.h
declares, and its host-side helpers (stream evaluation, workspace sizing,
argument validation) behave -- no kernel launches."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import pfr_oracle as O
from paper_1301_4019_b200 import _lib as L
from paper_1301_4019_b200.rng import RngStream, derive_seed

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1301_4019_b200 import _build

    _build.build()
    return L.load_library()


def _declared():
    src = open(os.path.join(ROOT, "include", "pfr.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|uint64_t|double|const char\*)\s+(pfr_\w+)\(", src, re.M)))


def test_exports_every_declared_symbol(lib):
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(L.exported_symbols()) == declared


def test_abi_version(lib):
    assert lib.pfr_abi_version() == 1


@pytest.mark.parametrize("seed,ids", [(0, ()), (1234, (5,)), (4242, (1, 2, 3)), (2**63 + 7, (9, 9))])
def test_numpy_stream_replay_on_host(lib, seed, ids):
    """pfr_stream_uniform(NUMPY) evaluates the same Philox4x64-10 code the
    kernels use; it must equal numpy's Generator.random() stream."""
    rs = RngStream(seed, ids)
    k0, k1 = rs.key()
    assert (k0, k1) == O.stream_key(seed, ids)
    want = O.generator(seed, ids).random(37)
    r = L.PfrRng(k0, k1, L.RNG_NUMPY, 0)
    got = np.array([lib.pfr_stream_uniform(r, i, 0) for i in range(37)])
    np.testing.assert_array_equal(got, want)


def test_philox4x32_known_answer(lib):
    """Own-stream draws equal the Random123 Philox4x32-10 restated in the oracle."""
    r = L.PfrRng(0x0123456789ABCDEF, 0, L.RNG_PHILOX, 0)
    for idx in (0, 1, 77, 2**33 + 5):
        o = O.philox4x32_10([idx & 0xFFFFFFFF, idx >> 32, 0x5359, 0], [0x89ABCDEF, 0x01234567])
        want = (((o[0] << 32) | o[1]) >> 11) * 2.0**-53
        assert lib.pfr_stream_uniform(r, idx, 0x5359) == want


def test_philox4x32_random123_vector():
    # Random123 kat_vectors: philox4x32_10 with all-ones counter/key
    ones = 0xFFFFFFFF
    assert O.philox4x32_10([ones] * 4, [ones] * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert O.philox4x32_10([0] * 4, [0] * 2) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]


def test_derive_seed_matches_oracle():
    for s, ids in [(0, ()), (42, (1, 2)), (2**64 - 1, (5,))]:
        assert derive_seed(s, *ids) == O.derive_seed(s, *ids)


def test_workspace_sizes(lib):
    for n in (1, 1000, 1 << 20):
        any_ = lib.pfr_workspace_bytes(L.OP_ANY, n, 0)
        assert any_ >= 28 * n
        assert lib.pfr_workspace_bytes(L.OP_SCAN, n, 0) < any_


def test_argument_validation_without_gpu(lib):
    rc = lib.pfr_scan(None, None, 0, L.F32, L.F32, 0, 0, None, None, None, 0, None)
    assert rc == L.E_ARG
    assert b"n must be" in lib.pfr_last_error()
    buf = ctypes.create_string_buffer(16)
    rc = lib.pfr_scan(ctypes.addressof(buf), ctypes.addressof(buf), 4, L.F64, L.F32, 0, 0, None, None, None, 0, None)
    assert rc == L.E_ARG  # float scans never narrow (float32 -> float64 widening is allowed)
    rc = lib.pfr_metropolis_range(ctypes.addressof(buf), 4, L.F32, 2, L.PfrRng(0, 0, 0, 0), 3, 2,
                                  ctypes.addressof(buf), None, None)
    assert rc == L.E_ARG and b"chain range" in lib.pfr_last_error()
    rc = lib.pfr_shard_offspring(ctypes.addressof(buf), 4, L.F32, 0.0, 0.0, 8, 0, 0, 0.5, None, None,
                                 ctypes.addressof(buf), None)
    assert rc == L.E_ARG and b"prefix/total" in lib.pfr_last_error()
    rc = lib.pfr_metropolis(ctypes.addressof(buf), 4, L.F32, -1, None, None, None, L.I64, ctypes.addressof(buf),
                            None, None, 0, None)
    assert rc == L.E_ARG and b"non-negative" in lib.pfr_last_error()
    rc = lib.pfr_rejection(ctypes.addressof(buf), 4, L.F32, 0.0, 0.0, L.PfrRng(0, 0, 0, 0), 10,
                           ctypes.addressof(buf), None, None, ctypes.addressof(buf), None, 0, None)
    assert rc == L.E_ARG and b"finite and positive" in lib.pfr_last_error()
    philox = L.PfrRng(0, 0, L.RNG_PHILOX, 0)
    rc = lib.pfr_rejection_range(ctypes.addressof(buf), 4, L.F32, 1.0, 0.0, philox, 10, 3, 2,
                                 ctypes.addressof(buf), None, None, ctypes.addressof(buf), None, 0, None)
    assert rc == L.E_ARG and b"slot range" in lib.pfr_last_error()
    rc = lib.pfr_rejection_range(ctypes.addressof(buf), 4, L.F32, 1.0, 0.0, L.PfrRng(0, 0, L.RNG_NUMPY, 0), 10, 0,
                                 2, ctypes.addressof(buf), None, None, ctypes.addressof(buf), None, 0, None)
    assert rc == L.E_ARG and b"PHILOX" in lib.pfr_last_error()
    rc = lib.pfr_probe_gather(ctypes.addressof(buf), 3, 4, 1, ctypes.addressof(buf), None)
    assert rc == L.E_ARG and b"power of two" in lib.pfr_last_error()
    rc = lib.pfr_probe_gather(ctypes.addressof(buf), 4, 2, 1, ctypes.addressof(buf), None)
    assert rc == L.E_ARG and b"elem_bytes" in lib.pfr_last_error()


def test_host_scalars():
    import paper_1301_4019_b200 as pf

    assert pf.metropolis_num_steps(0.5, 0.005, 16) == 35
    assert pf.metropolis_num_steps(1.0, 0.01, 4) == 17
    assert pf.metropolis_num_steps(0.5, None, 16) == 35
    with pytest.raises(ValueError, match="p_star.*too small|bias bound"):
        pf.metropolis_num_steps(0.01, 0.0001, 16)
    with pytest.raises(ValueError):
        pf.metropolis_num_steps(0.5, 0.6, 16)
    assert pf.stratum_offset_kernel(2.0**24, 0.25, 2**25, np.float32) == 2**24
    assert pf.stratum_offset_kernel(float(2**23), 0.75, 2**23, np.float32) == 2**23
    assert pf.stratum_offset_kernel(3.7, 0.5, 100) == 4
    with pytest.raises(ValueError):
        pf.ResamplerConfig(algorithm="residual")


def test_product_path_refuses_without_gpu():
    import torch

    import paper_1301_4019_b200 as pf

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA device"):
        pf.inclusive_prefix_sum([1.0, 2.0])
