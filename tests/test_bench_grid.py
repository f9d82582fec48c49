"""The GPU benchmark grid: the reference's CSV schema,
its weight sets draw for draw, the CLI, error markers."""

from __future__ import annotations

import numpy as np
import pytest
from click.testing import CliRunner

from paper_1301_4019_b200 import bench_grid as B
from paper_1301_4019_b200.__main__ import _parse_float_list, _parse_int_list, main


def test_grid_parsing_and_config():
    assert _parse_int_list("2^4..2^6,100") == (16, 32, 64, 100)
    assert _parse_float_list("0..1:0.5,3") == (0.0, 0.5, 1.0, 3.0)
    with pytest.raises(ValueError):
        B.BenchConfig(algorithms=("bogus",))
    cfg = B.BenchConfig(algorithms=("systematic",), n_values=(16,), y_values=(0.0, 1.0), replicates=2)
    assert len(list(cfg.cells())) == 4


def test_weight_sets_match_the_reference_recipe():
    w = B.simulate_weight_set(B.WeightSetSpec(64, 1.0, 7))
    assert w.shape == (64,) and np.all(w > 0) and np.all(w <= B.sup_weight())
    assert B.max_normalised_weight(0.0, 1) == 1.0
    assert B.expected_weight(0.0) == pytest.approx(1 / (2 * np.sqrt(np.pi)))


def test_csv_round_trip(tmp_path):
    recs = [B.BenchRecord("systematic", 16, 0.5, 0, 1234, 0.001, {"gbps": 1.5}),
            B.BenchRecord("metropolis", 16, 0.5, 1, 0, None, {"error": "x"})]
    p = tmp_path / "r.csv"
    B.write_records_csv(recs, p)
    back = B.read_records_csv(p)
    assert [r.sort_key() for r in back] == [r.sort_key() for r in recs]
    assert back[1].mse is None and open(p).readline().strip() == ",".join(B.CSV_COLUMNS)


@pytest.mark.gpu
def test_grid_runs_every_algorithm(tmp_path):
    out = tmp_path / "grid.csv"
    res = CliRunner().invoke(main, ["bench", "run", "--n", "2^6,2^10", "--y", "0..2:1", "--reps", "2",
                                    "--out", str(out)])
    assert res.exit_code == 0, res.output
    recs = B.read_records_csv(out)
    assert len(recs) == 7 * 2 * 3 * 2 and all(r.mse is not None for r in recs)
    rows = B.aggregate_rmse(recs)
    assert len(rows) == 7 * 2 * 3 and all(r[4] >= 0 for r in rows)
    agg = tmp_path / "rmse.csv"
    res = CliRunner().invoke(main, ["bench", "aggregate", "--in", str(out), "--out", str(agg)])
    assert res.exit_code == 0, res.output


@pytest.mark.gpu
def test_grid_is_deterministic_across_workers_and_runs():
    """SPEC C11 (test_acceptance.py:350-388): the same grid twice, with 1 and
    4 workers, gives identical records except the timing columns."""
    cfg1 = B.BenchConfig(n_values=(64, 1024), y_values=(0.0, 2.0), replicates=2, workers=1)
    cfg4 = B.BenchConfig(n_values=(64, 1024), y_values=(0.0, 2.0), replicates=2, workers=4)
    r1, e1 = B.run_grid(cfg1)
    r4, e4 = B.run_grid(cfg4)
    assert e1 == e4 == 0
    key = lambda r: (r.algorithm, r.n, r.y, r.replicate, r.mse,  # noqa: E731
                     {k: v for k, v in r.extras.items() if k != "gbps"})
    assert [key(r) for r in r1] == [key(r) for r in r4]
