"""stable_sum, permute_serial, ESS and resampling MSE (the remaining reference
functions around the step).  CPU: the oracle restatements against golden
vectors produced by the reference.  GPU: the kernels against the same
fixtures (stable_sum bit for bit: the pairwise tree's association is fixed)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import pfr_oracle as O
from tests.golden.make_golden import ANCESTRY_CASES, STABLE_CASES, golden_ancestry, stable_vector


@pytest.mark.parametrize("k", range(len(STABLE_CASES)))
def test_oracle_stable_sum(golden, k):
    v = stable_vector(k)
    assert np.float64(v.astype(np.float64).sum()) == golden[f"stable/{k}/checksum"]
    assert O.stable_sum(v) == golden[f"stable/{k}/sum"]


@pytest.mark.parametrize("k", range(3))
def test_oracle_weight_stats(golden, k):
    w, o = golden[f"wstats/{k}/w"], golden[f"wstats/{k}/o"]
    assert O.ess(w) == golden[f"wstats/{k}/ess"]
    assert O.resampling_mse(o, w) == golden[f"wstats/{k}/mse"]


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(STABLE_CASES)))
def test_stable_sum_bit_exact(golden, k):
    import paper_1301_4019_b200 as pf

    got = pf.stable_sum(stable_vector(k))
    want = golden[f"stable/{k}/sum"]
    assert got.dtype == want.dtype and got == want, (got, want)


@pytest.mark.gpu
def test_stable_sum_kats():
    import paper_1301_4019_b200 as pf

    assert pf.stable_sum([1.0, 2.0, 3.0, 4.0]) == 10.0
    assert pf.stable_sum([3.25]) == 3.25
    w = np.concatenate(([2.0 ** 24], np.ones(4096))).astype(np.float32)
    stable = pf.stable_sum(w)
    naive = pf.vector_sum(w)
    exact = 2.0 ** 24 + 4096
    assert float(stable) >= float(naive)
    assert abs(float(stable) - exact) <= abs(float(naive) - exact)
    with pytest.raises(ValueError, match="finite"):
        pf.stable_sum([1.0, np.nan])


@pytest.mark.gpu
@pytest.mark.parametrize("n,seed", ANCESTRY_CASES)
@pytest.mark.parametrize("sorted_", [False, True])
def test_permute_serial_golden(golden, n, seed, sorted_):
    import paper_1301_4019_b200 as pf

    a = golden_ancestry(n, seed, sorted_)
    tag = f"anc{n}_{'s' if sorted_ else 'u'}"
    c = pf.permute_serial(a).cpu().numpy()
    np.testing.assert_array_equal(c, golden[f"{tag}/serial"])


@pytest.mark.gpu
def test_permute_serial_kat():
    import paper_1301_4019_b200 as pf

    np.testing.assert_array_equal(pf.permute_serial([2, 0, 0]).cpu().numpy(), [0, 0, 2])


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(3))
def test_weight_stats_against_reference(golden, k):
    import paper_1301_4019_b200 as pf

    w, o = golden[f"wstats/{k}/w"], golden[f"wstats/{k}/o"]
    assert pf.ess(w) == pytest.approx(float(golden[f"wstats/{k}/ess"]), rel=1e-13)
    assert pf.resampling_mse(o, w) == pytest.approx(float(golden[f"wstats/{k}/mse"]), rel=1e-11)


@pytest.mark.gpu
def test_weight_stats_kats():
    import paper_1301_4019_b200 as pf

    assert pf.resampling_mse(np.ones(8, dtype=int), np.full(8, 0.3)) == 0.0
    assert pf.resampling_mse([2, 0], [1.0, 1.0]) == pytest.approx(0.25)
    with pytest.raises(ValueError):
        pf.resampling_mse([1, 1], [1.0, 1.0, 1.0])
    assert pf.ess(np.ones(100)) == pytest.approx(100.0)
    assert pf.ess([0.0, 0.0, 3.0]) == pytest.approx(1.0)


@pytest.mark.gpu
def test_ctypes_example_without_torch():
    """examples/ctypes_deliver.py: the C ABI driven through ctypes and
    cuda-python only (the FFI path of a non-Python host)."""
    import subprocess
    import sys

    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(os.path.dirname(__file__)), "examples",
                                                     "ctypes_deliver.py"), "100003"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
    assert "hold" in r.stdout


@pytest.mark.gpu
def test_c_example_compiles_and_runs(tmp_path):
    """examples/deliver.c: include/pfr.h is plain C; a C host links
    libpfr.so and runs a fused delivery."""
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_1301_4019_b200")
    exe = str(tmp_path / "deliver")
    cc = subprocess.run(["gcc", "-std=c11", "-Wall", "-I", os.path.join(root, "include"), "-I",
                         "/usr/local/cuda/include", os.path.join(root, "examples", "deliver.c"), "-L", libdir,
                         "-lpfr", "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{libdir}",
                         "-Wl,-rpath,/usr/local/cuda/lib64", "-o", exe], capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr
    r = subprocess.run([exe, "300007"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "holds" in r.stdout


@pytest.mark.gpu
def test_graft_entry_smoke():
    """__graft_entry__.smoke(): one small delivery + Metropolis on cuda:0,
    checked against the oracle (the driver runs it at round end)."""
    import importlib
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    entry = importlib.import_module("__graft_entry__")
    entry.smoke()
