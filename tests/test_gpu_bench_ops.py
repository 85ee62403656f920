"""GPU bench-ops: the reference's report schema
(cli.py:279-306) plus device time / bytes / roofline fraction."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("batch", [1, 4])
def test_bench_ops_schema(batch):
    from paper_2310_16530_b200 import bench_ops
    rep = bench_ops.run("unit", reps=3, seed=0, batch=batch)
    assert rep["command"] == "bench-ops" and rep["version"] == 1 and rep["params"] == "unit"
    assert set(rep["ops"]) == set(bench_ops.BENCH_OPS)
    for name, r in rep["ops"].items():
        assert r["median_ms"] > 0 and r["device_ms"] > 0 and r["algorithmic_bytes"] > 0
        assert 0 < r["roofline_frac"] < 2
    assert rep["hmult_gt_hadd"] is True
