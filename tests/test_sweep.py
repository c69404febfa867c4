"""N / l / k sweep harness (paper_2105_12026_b200/sweep.py, the reference's
bench.py:21-186) and the CLI ``bench`` subcommand (cli.py:252-267, 330-342)."""

import os
import sys

import numpy as np
import pytest

from paper_2105_12026_b200 import cli, sweep
from paper_2105_12026_b200.core import Precision

REF_SRC = "/root/reference/pkg/src"


def test_problem_spec_validation_and_axes():
    with pytest.raises(ValueError, match="k=6 exceeds n=5"):
        sweep.ProblemSpec(n=5, l=1, k=6, dims=2)
    with pytest.raises(ValueError, match="dims must be >= 1"):
        sweep.ProblemSpec(n=5, l=1, k=1, dims=0)
    s = sweep.ProblemSpec(n=100, l=7, k=3, dims=4, seed=9)
    assert s.with_axis("N", 200).n == 200 and s.with_axis("l", 9).l == 9 and s.with_axis("k", 5).k == 5
    assert sweep.DEFAULT_AXIS_VALUES["N"][0] == 1000 and sweep.DEFAULT_AXIS_VALUES["k"][-1] == 430


def test_generate_problem_is_a_pure_function_of_the_spec():
    spec = sweep.ProblemSpec(n=300, l=12, k=4, dims=5, seed=3, precision=Precision.FP32)
    g1, m1 = sweep.generate_problem(spec)
    g2, m2 = sweep.generate_problem(spec)
    np.testing.assert_array_equal(g1.data, g2.data)
    assert m1.sets == m2.sets and len(m1.sets) == 12
    assert all(len(set(s)) == 4 for s in m1.sets)
    rng = np.random.default_rng(3)  # bench.py:58-62: cells first, then the sets
    np.testing.assert_array_equal(g1.data, rng.random((300, 5)).astype(np.float32))


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present (GPU box)")
def test_generate_problem_matches_reference():
    sys.path.insert(0, REF_SRC)
    try:
        from ebcsum import bench as rb
        from ebcsum.core import Precision as RP
    finally:
        sys.path.remove(REF_SRC)
    for prec, rprec in ((Precision.FP32, RP.FP32), (Precision.FP16_STORAGE, RP.FP16_STORAGE)):
        ours = sweep.generate_problem(sweep.ProblemSpec(n=257, l=9, k=6, dims=7, seed=11, precision=prec))
        ref = rb.generate_problem(rb.ProblemSpec(n=257, l=9, k=6, dims=7, seed=11, precision=rprec))
        np.testing.assert_array_equal(ours[0].data, ref[0].data)
        assert ours[1].sets == ref[1].sets


def _report():
    r = sweep.SweepReport(axis="l", values=[10, 20], backends=["b200", "b200:2"], repeats=2)
    r.runtimes = {(10, "b200"): [1.0, 2.0], (10, "b200:2"): [0.5, 1.0],
                  (20, "b200"): [4.0, 4.0], (20, "b200:2"): [2.0, 1.0]}
    r.comparisons = sweep.aggregate_speedups(r)
    return r


def test_speedups_and_reports():
    r = _report()
    c = {(x.baseline, x.subject): x for x in r.comparisons}
    assert c[("b200", "b200:2")].min == 2.0 and c[("b200", "b200:2")].max == 4.0
    assert c[("b200", "b200")].mean == 1.0
    csv_text = sweep.emit_report(r, "csv")
    assert csv_text.splitlines()[0] == "axis,value,backend,run,runtime_seconds"
    assert "l,20,b200:2,1,1.000000000" in csv_text
    assert "b200,b200:2,2.000000,2.500000,4.000000" in csv_text
    md = sweep.emit_report(r, "markdown")
    assert "| 10 | 1.500000 s | 0.750000 s |" in md and "| b200 | b200:2 | 2.000x | 2.500x | 4.000x |" in md
    with pytest.raises(ValueError, match="unknown report format"):
        sweep.emit_report(r, "xml")
    with pytest.raises(ValueError, match="no measurements"):
        sweep.emit_report(sweep.SweepReport("N", [], [], 1), "csv")


def test_run_sweep_validates_before_touching_the_device():
    base = sweep.ProblemSpec(n=50, l=5, k=2, dims=3)
    with pytest.raises(ValueError, match="axis must be one of"):
        sweep.run_sweep("d", [1], base, ["b200"])
    with pytest.raises(ValueError, match="sorted ascending"):
        sweep.run_sweep("l", [9, 3], base, ["b200"])
    with pytest.raises(ValueError, match="repeats must be >= 1"):
        sweep.run_sweep("l", [3], base, ["b200"], repeats=0)
    with pytest.raises(ValueError, match="unknown backend"):
        sweep.run_sweep("l", [3], base, ["batched:4"])
    with pytest.raises(ValueError, match="thread count"):
        sweep.run_sweep("l", [3], base, ["ref-batched:0"])


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present (GPU box)")
def test_run_sweep_reference_cpu_columns(monkeypatch):
    """The CPU baseline columns run the reference package's own backends."""
    monkeypatch.setenv("EBCSUM_PATH", REF_SRC)
    base = sweep.ProblemSpec(n=300, l=8, k=3, dims=4, seed=1)
    rep = sweep.run_sweep("l", [4, 8], base, ["ref-naive", "ref-batched:2"], repeats=2)
    assert rep.backends == ["ref-naive", "ref-batched:2"]
    assert all(len(rep.runtimes[(v, b)]) == 2 for v in (4, 8) for b in rep.backends)
    c = {(x.baseline, x.subject): x for x in rep.comparisons}
    assert c[("ref-naive", "ref-naive")].mean == 1.0


def test_cli_bench_exit_codes(capsys):
    assert cli.main(["bench", "--values", "x,1"]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--axis", "l", "--values", "9,3", "--n", "50", "--l", "5", "-k", "2",
                     "--dims", "3"]) == cli.EXIT_DATA
    assert "sorted ascending" in capsys.readouterr().err


@pytest.mark.gpu
def test_run_sweep_on_the_device(tmp_path):
    base = sweep.ProblemSpec(n=600, l=16, k=4, dims=8, seed=2)
    cols = ["b200", "b200:4"] + (["ref-batched:2"] if sweep._reference_package() is not None else [])
    rep = sweep.run_sweep("l", [8, 16], base, cols, repeats=2)
    assert set(rep.runtimes) == {(v, b) for v in (8, 16) for b in cols}
    assert all(len(v) == 2 and min(v) > 0 for v in rep.runtimes.values())
    out = tmp_path / "sweep.md"
    assert cli.main(["bench", "--axis", "k", "--values", "2,5", "--n", "400", "--l", "20", "--dims", "6",
                     "--repeats", "2", "--format", "markdown", "--output", str(out)]) == cli.EXIT_OK
    assert out.read_text().startswith("## Sweep over k (2 runs per value)")
