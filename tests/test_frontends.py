"""Host-side logic of the thin wrappers -- CPU only:
GenSpec draws against the reference's digests, file parsing and its errors,
the CLI's usage / error exit codes and the estimator's sklearn protocol."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2202_07258_b200.errors import BadSpec, DimensionMismatch, ParseError, ZeroColumn, ZeroRow
from paper_2202_07258_b200.generate import GenSpec, generate

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _digest(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_genspec_draws_match_reference():
    """generate.py:39-77 restated: identical arrays for the same spec."""
    z = np.load(os.path.join(GOLD, "frontends.npz"))
    for text, dig in zip(z["gen_specs"], z["gen_digest"]):
        p = generate(GenSpec(**json.loads(str(text))))
        assert _digest(p.a_matrix, p.y, p.lower, p.upper) == str(dig), text


def test_genspec_validation():
    for bad in (dict(family="x", m=3, n=3), dict(family="nnls", m=0, n=3),
                dict(family="bvls", m=3, n=3, box_halfwidth=0.0), dict(family="nnls", m=3, n=3, sparsity=0.0),
                dict(family="nnls", m=3, n=4, sparsity=0.1)):
        with pytest.raises(BadSpec):
            GenSpec(**bad)


def test_instance_hash_matches_reference():
    from paper_2202_07258_b200.bench import instance_hash
    z = np.load(os.path.join(GOLD, "frontends.npz"))
    for text, h in zip(z["gen_specs"], z["gen_instance_hash"]):
        assert instance_hash(generate(GenSpec(**json.loads(str(text))))) == str(h)


def test_parsing_errors(tmp_path):
    from paper_2202_07258_b200.problem_io import load_problem, parse_bounds, read_csv_array
    f = tmp_path / "a.csv"
    f.write_text("1,2\n3,x\n")
    with pytest.raises(ParseError, match="line 2, column 2"):
        read_csv_array(f)
    f.write_text("1,2\n3\n")
    with pytest.raises(ParseError, match="ragged"):
        read_csv_array(f)
    f.write_text("\n\n")
    with pytest.raises(ParseError, match="empty"):
        read_csv_array(f)
    f.write_text("1,2\n")
    with pytest.raises(ParseError, match="expected 1 fields"):
        read_csv_array(f, ncols=1)
    lo, hi = parse_bounds("box:-1:2", 3)
    assert lo.tolist() == [-1.0] * 3 and hi.tolist() == [2.0] * 3
    lo, hi = parse_bounds("nn", 2)
    assert np.isinf(hi).all() and (lo == 0).all()
    for spec in ("box:1", "box:a:b", "nope"):
        with pytest.raises(ParseError):
            parse_bounds(spec, 2)
    b = tmp_path / "b.csv"
    b.write_text("0,inf\n-1,1\n")
    lo, hi = parse_bounds(str(b), 2)
    assert lo.tolist() == [0.0, -1.0] and hi[0] == np.inf and hi[1] == 1.0
    with pytest.raises(DimensionMismatch):
        parse_bounds(str(b), 3)
    # zero column / zero row / y length (host path)
    a = tmp_path / "m.csv"
    y = tmp_path / "y.csv"
    a.write_text("1,0\n2,0\n")
    y.write_text("1\n2\n")
    with pytest.raises(ZeroColumn):
        load_problem(a, y, "nn", device=None)
    a.write_text("1,2\n0,0\n")
    with pytest.raises(ZeroRow):
        load_problem(a, y, "nn", device=None)
    y.write_text("1\n2\n3\n")
    with pytest.raises(DimensionMismatch):
        load_problem(a, y, "nn", device=None)


def test_save_load_round_trip(tmp_path):
    from paper_2202_07258_b200.problem_io import load_problem, save_problem
    p = generate(GenSpec(family="bvls", m=7, n=5, box_halfwidth=0.5, seed=3))
    pa, py, pb = save_problem(p, str(tmp_path / "q"))
    q = load_problem(pa, py, pb, device=None)
    np.testing.assert_array_equal(q.a_matrix, p.a_matrix)
    np.testing.assert_array_equal(q.y, p.y)
    np.testing.assert_array_equal(q.upper, p.upper)
    qn = load_problem(pa, py, "box:-0.5:0.5", normalize_columns=True, device=None)
    np.testing.assert_allclose(np.linalg.norm(qn.a_matrix, axis=0), 1.0)


def test_cli_usage_and_error_codes(tmp_path, capsys):
    from paper_2202_07258_b200.cli import cli_main
    assert cli_main([]) == 1                       # argparse usage error
    assert cli_main(["solve"]) == 1                # missing required flags
    assert cli_main(["--help"]) == 0
    bad = tmp_path / "bad.csv"
    bad.write_text("1,x\n")
    y = tmp_path / "y.csv"
    y.write_text("1\n")
    assert cli_main(["solve", "--a", str(bad), "--y", str(y)]) == 2
    assert "ParseError" in capsys.readouterr().err
    assert cli_main(["gen", "--family", "nnls", "--m", "5", "--n", "4", "--sparsity", "0.1",
                     "--out-prefix", str(tmp_path / "g")]) == 2   # BadSpec
    assert cli_main(["gen", "--family", "nnls", "--m", "6", "--n", "20", "--seed", "1",
                     "--out-prefix", str(tmp_path / "g")]) == 0
    from paper_2202_07258_b200.problem_io import load_problem
    q = load_problem(tmp_path / "g_A.mtx", tmp_path / "g_y.csv", str(tmp_path / "g_bounds.csv"), device=None)
    p = generate(GenSpec(family="nnls", m=6, n=20, seed=1))
    np.testing.assert_array_equal(q.a_matrix, p.a_matrix)
    np.testing.assert_array_equal(q.y, p.y)


def test_estimator_params_and_unfitted():
    from sklearn.exceptions import NotFittedError
    from paper_2202_07258_b200.estimator import BoxConstrainedRegression
    est = BoxConstrainedRegression(solver="pg", tol=1e-7)
    assert est.get_params()["solver"] == "pg"
    est.set_params(solver="active-set")
    assert est.solver == "active-set"
    with pytest.raises(NotFittedError):
        BoxConstrainedRegression().predict(np.eye(3))
