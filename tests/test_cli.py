"""CLI front end (paper_2105_12026_b200/cli.py): the reference's summarize
contract (cli.py:59-108, 229-327) -- CSV parsing errors, normalisation, exit
codes, JSON document -- and the surrogate writer."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2105_12026_b200 import cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _write(tmp_path, text, name="d.csv"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_load_csv_header_blank_lines_and_normalize(tmp_path):
    p = _write(tmp_path, "a,b,c\n1,2,5\n\n3,2,7\n")
    data, header = cli.load_csv(p, has_header=True)
    assert header == ["a", "b", "c"]
    np.testing.assert_array_equal(data, [[1, 2, 5], [3, 2, 7]])
    z, _ = cli.load_csv(p, has_header=True, normalize=True)
    np.testing.assert_allclose(z, [[-1, 0, -1], [1, 0, 1]])  # constant column stays 0


@pytest.mark.parametrize("text, msg", [
    ("1,2\n3\n", "row 2: expected 2 columns, got 1"),
    ("1,x\n", "row 1, column 2: not a number: 'x'"),
    ("1,inf\n", "row 1, column 2: non-finite value 'inf'"),
    ("\n\n", "no data rows"),
])
def test_load_csv_errors_name_row_and_column(tmp_path, text, msg):
    with pytest.raises(cli.CsvParseError, match=msg):
        cli.load_csv(_write(tmp_path, text))


def test_exit_codes_usage_and_data(tmp_path, capsys):
    assert cli.main(["summarize", "x.csv"]) == cli.EXIT_USAGE  # -k missing
    assert cli.main(["summarize", "x.csv", "-k", "0"]) == cli.EXIT_USAGE
    assert cli.main(["summarize", str(tmp_path / "missing.csv"), "-k", "1"]) == cli.EXIT_DATA
    assert cli.main(["summarize", _write(tmp_path, "1,x\n"), "-k", "1"]) == cli.EXIT_DATA
    assert cli.main(["surrogate", "--cycles", "10", "--regimes", "3", "--output", str(tmp_path / "s.csv")]) \
        == cli.EXIT_DATA


def test_surrogate_writer_matches_generator(tmp_path):
    from paper_2105_12026_b200.surrogate import surrogate
    out = tmp_path / "s.csv"
    assert cli.main(["surrogate", "--cycles", "50", "--dims", "8", "--cycles-per-regime", "10",
                     "--output", str(out)]) == cli.EXIT_OK
    data, _ = cli.load_csv(str(out))
    np.testing.assert_array_equal(data, surrogate(50, 8, 5, 0.01, 0))
    # the regime-label sidecar (reference cli.py:176-187): stem + "_labels"
    lab = np.loadtxt(tmp_path / "s_labels.csv", dtype=np.int64)
    np.testing.assert_array_equal(lab, np.repeat(np.arange(5), 10))


def test_surrogate_spec_contract(tmp_path, capsys):
    """SurrogateSpec validation (reference cli.py:121-131): the default
    --cycles-per-regime is 200, so --cycles 1000 --regimes 5 is the default case
    and any product mismatch is a data error naming both sides."""
    out = str(tmp_path / "d.csv")
    assert cli.main(["surrogate", "--dims", "4", "--output", out]) == cli.EXIT_OK
    assert np.loadtxt(out, delimiter=",").shape == (1000, 4)
    assert cli.main(["surrogate", "--cycles", "100", "--regimes", "5", "--output", out]) == cli.EXIT_DATA
    assert "n_regimes * cycles_per_regime must equal n_cycles (5 * 200 != 100)" in capsys.readouterr().err
    assert cli.main(["surrogate", "--noise", "-1", "--output", out]) == cli.EXIT_DATA


def test_summarize_accepts_reference_threads_flag():
    """--threads (reference cli.py:247) parses; the device path ignores it."""
    args = cli.build_parser().parse_args(["summarize", "x.csv", "-k", "2", "--threads", "4"])
    assert args.threads == 4
    assert cli.main(["summarize", "x.csv", "-k", "2", "--threads", "0"]) == cli.EXIT_USAGE


@pytest.mark.gpu
@pytest.mark.parametrize("optimizer", ["greedy", "sieve"])
def test_summarize_on_gpu_matches_oracle(tmp_path, optimizer):
    import oracle
    import paper_2105_12026_b200 as eb
    X = np.random.default_rng(3).standard_normal((400, 6))
    p = tmp_path / "x.csv"
    np.savetxt(p, X, delimiter=",", fmt="%.17g")
    out = tmp_path / "o.json"
    r = subprocess.run([sys.executable, "-m", "paper_2105_12026_b200", "summarize", str(p), "-k", "5",
                        "--optimizer", optimizer, "--output", str(out)], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    doc = json.loads(out.read_text())
    assert doc["precision"] == "fp64" and doc["backend"] == "b200" and doc["k"] == 5
    if optimizer == "greedy":
        sel, vals, _, _ = oracle.greedy(X, 5)
        assert doc["selected_indices"] == sel
        assert doc["function_value"] == pytest.approx(vals[-1], rel=1e-12)
    else:
        f = eb.EbcFunction(eb.GroundMatrix(X))
        s = eb.sieve_stream_maximize(np.random.default_rng(0).permutation(400), f, 5, epsilon=0.1)
        assert doc["selected_indices"] == s.selected
