"""The thin wrappers around the GPU solver against the
REAL reference's outputs (tests/golden/frontends.npz): estimator fits,
compare_t curves, solve-linear translation vectors, the CLI's solve result,
device-side problem ingestion and the benchmark runner."""

import csv
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _z():
    return np.load(os.path.join(GOLD, "frontends.npz"))


def _obj(a, y, x):
    r = a @ x - y
    return 0.5 * float(r @ r)


def test_estimator_fits_vs_reference():
    """test_estimator.py shapes: same coefficients (1e-8), rounds and
    convergence as the reference's BoxConstrainedRegression."""
    from paper_2202_07258_b200.estimator import BoxConstrainedRegression
    from paper_2202_07258_b200.generate import GenSpec, generate
    z = _z()
    for name in z["fit_names"]:
        name = str(name)
        kw = json.loads(str(z[f"fit_{name}_kw"]))
        p = generate(GenSpec(**json.loads(str(z[f"fit_{name}_spec"]))))
        est = BoxConstrainedRegression(**kw).fit(p.a_matrix, p.y)
        ref = z[f"fit_{name}_coef"]
        assert np.max(np.abs(est.coef_ - ref)) <= 1e-8 * max(1.0, np.max(np.abs(ref))), name
        gap, n_iter, conv = z[f"fit_{name}_stats"]
        assert est.n_iter_ == int(n_iter) and est.converged_ == bool(conv), name
        assert len(est.trace_) == est.n_iter_
        assert est.n_features_in_ == p.n
        np.testing.assert_allclose(est.predict(p.a_matrix), p.a_matrix @ est.coef_)


def test_estimator_screening_off_and_bounds():
    from paper_2202_07258_b200.estimator import BoxConstrainedRegression
    from paper_2202_07258_b200.generate import GenSpec, generate
    p = generate(GenSpec(family="nnls", m=30, n=20, seed=2))
    on = BoxConstrainedRegression(tol=1e-8).fit(p.a_matrix, p.y)
    off = BoxConstrainedRegression(tol=1e-8, screening=False).fit(p.a_matrix, p.y)
    o_on, o_off = _obj(p.a_matrix, p.y, on.coef_), _obj(p.a_matrix, p.y, off.coef_)
    assert abs(o_on - o_off) <= 1e-8 * max(1.0, o_off)
    b = generate(GenSpec(family="bvls", m=25, n=10, box_halfwidth=0.4, seed=1))
    for solver in ("pg", "cd", "apg", "active-set"):
        est = BoxConstrainedRegression(lower=-0.4, upper=0.4, solver=solver).fit(b.a_matrix, b.y)
        assert est.converged_ and np.all(est.coef_ >= -0.4) and np.all(est.coef_ <= 0.4), solver


def test_compare_t_vs_reference():
    """test_harness.py:221-229: three strategies, curves on a common grid,
    each monotone, equal to the reference's screening ratios."""
    from paper_2202_07258_b200.bench import compare_t
    from paper_2202_07258_b200.generate import GenSpec, generate
    z = _z()
    p = generate(GenSpec(family="nnls", m=30, n=40, seed=2))
    rounds, curves = compare_t(p, ["neg-ones", "neg-mean-column", ("neg-column", {"column": 0})])
    assert list(curves) == [str(s) for s in z["ct_labels"]]
    assert rounds == list(range(1, z["ct_curves"].shape[1] + 1))
    for i, (label, c) in enumerate(curves.items()):
        assert all(a <= b for a, b in zip(c, c[1:])), label
        np.testing.assert_array_equal(c, z["ct_curves"][i], err_msg=label)


def test_translation_vectors():
    """solve-linear (device Cholesky) vs the reference's t; construction-time
    interiority check and the rank-deficient failure (test_duality.py:221-264)."""
    from paper_2202_07258_b200 import Problem, select_translation_vector
    from paper_2202_07258_b200.errors import NoInteriorPoint, SingularGram
    z = _z()
    p = Problem(z["sl_a"], z["sl_y"], 0.0, np.inf)
    tv = select_translation_vector(p, "solve-linear")
    np.testing.assert_allclose(tv.t, z["sl_t"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(tv.a_t_t, p.a_matrix.T @ tv.t, rtol=1e-12, atol=1e-12)
    assert np.all(tv.a_t_t < 0)
    rng = np.random.default_rng(1)
    wide = Problem(np.abs(rng.standard_normal((3, 6))), rng.standard_normal(3), 0.0, np.inf)
    with pytest.raises((SingularGram, NoInteriorPoint)):
        select_translation_vector(wide, "solve-linear")
    # a column orthogonal to t = -a_0 is not strictly interior
    a = np.array([[1.0, 0.0], [0.0, 1.0]])
    with pytest.raises(NoInteriorPoint):
        select_translation_vector(Problem(a, [1.0, 1.0], 0.0, np.inf), "neg-column", column=0)
    ok = select_translation_vector(Problem(np.abs(rng.standard_normal((5, 4))) + 0.1, np.ones(5), 0.0, np.inf),
                                   "neg-mean-column")
    assert np.all(ok.a_t_t < 0)


def test_cli_solve_vs_reference(tmp_path):
    """`gen` + `solve` through the CLI: the result JSON's x / gap / rounds
    against the reference CLI's on the same files; trace CSV header."""
    from paper_2202_07258_b200.cli import cli_main
    z = _z()
    pre = str(tmp_path / "p")
    assert cli_main(["gen", "--family", "nnls", "--m", "40", "--n", "60", "--seed", "5", "--out-prefix", pre]) == 0
    rj, tc = str(tmp_path / "r.json"), str(tmp_path / "t.csv")
    assert cli_main(["solve", "--a", pre + "_A.mtx", "--y", pre + "_y.csv", "--solver", "pg", "--inner-passes", "5",
                     "--tol", "1e-8", "--result-out", rj, "--trace-out", tc]) == 0
    with open(rj) as fh:
        r = json.load(fh)
    x_ref = z["cli_x"]
    assert np.max(np.abs(np.array(r["x"]) - x_ref)) <= 1e-8 * max(1.0, np.max(np.abs(x_ref)))
    gap, rounds, conv = z["cli_stats"]
    assert r["rounds"] == int(rounds) and r["converged"] == bool(conv)
    with open(tc) as fh:
        rows = list(csv.reader(fh))
    assert ",".join(rows[0]) == str(z["cli_trace_header"])
    assert len(rows) == int(rounds) + 1
    # a NoInteriorPoint from the translation vector is exit code 2
    tfile = tmp_path / "t.csv"
    tfile.write_text("1\n" * 40)
    assert cli_main(["solve", "--a", pre + "_A.mtx", "--y", pre + "_y.csv", "--t-strategy", f"custom={tfile}"]) == 2
    # compare-t writes one column per strategy
    out = str(tmp_path / "ct.csv")
    assert cli_main(["compare-t", "--gen-m", "30", "--gen-n", "40", "--seed", "2", "--out", out]) == 0
    with open(out) as fh:
        assert next(csv.reader(fh)) == ["round", "neg-ones", "neg-mean-column"]


def test_device_ingestion(tmp_path):
    """load_problem straight into device buffers: norms, zero row / column
    rejection and column normalisation on the GPU; same solve as the host path."""
    import torch
    from paper_2202_07258_b200 import SolverConfig, solve
    from paper_2202_07258_b200.errors import ZeroColumn, ZeroRow
    from paper_2202_07258_b200.generate import GenSpec, generate
    from paper_2202_07258_b200.problem_io import load_problem, save_problem
    p = generate(GenSpec(family="nnls", m=40, n=60, seed=4))
    pa, py, pb = save_problem(p, str(tmp_path / "q"))
    qd = load_problem(pa, py, "nn", normalize_columns=True, device="cuda")
    qh = load_problem(pa, py, "nn", normalize_columns=True, device=None)
    assert qd.a_matrix is None and qd.device_arrays()["a"].is_cuda
    cfg = SolverConfig(kind="cd", gap_tol=1e-9)
    rd, rh = solve(qd, cfg), solve(qh, cfg)
    assert rd.rounds == rh.rounds
    np.testing.assert_allclose(rd.x, rh.x, rtol=1e-9, atol=1e-12)
    a = tmp_path / "z.csv"
    y = tmp_path / "y.csv"
    a.write_text("1,0\n2,0\n")
    y.write_text("1\n2\n")
    with pytest.raises(ZeroColumn):
        load_problem(a, y, "nn", device="cuda")
    a.write_text("1,2\n0,0\n")
    with pytest.raises(ZeroRow):
        load_problem(a, y, "nn", device="cuda")
    del torch


def test_run_bench_sweep(tmp_path):
    """Paired off / on cells; an error cell does not abort the sweep
    (test_harness.py:195-213)."""
    from paper_2202_07258_b200.bench import run_bench
    from paper_2202_07258_b200.generate import GenSpec
    rep = run_bench([GenSpec(family="nnls", m=15, n=20, seed=0), GenSpec(family="bvls", m=12, n=8, seed=1)],
                    ["cd", "pg"], repetitions=2)
    assert len(rep.rows) == 8 and len(rep.speedups) == 4
    for s in rep.speedups:
        assert s["elapsed_on"] > 0 and s["elapsed_off"] > 0
    rep.rows_to_csv(tmp_path / "rows.csv")
    rep.speedups_to_csv(tmp_path / "sp.csv")
    assert json.loads(rep.to_json(tmp_path / "r.json"))["meta"]["repetitions"] == 2
    mixed = run_bench([GenSpec(family="nnls", m=15, n=20, seed=0)], ["cd", "bogus"], repetitions=1)
    assert len(mixed.speedups) == 1 and len(mixed.meta["errors"]) == 1
    assert "ValueError" in mixed.meta["errors"][0]["error"]
