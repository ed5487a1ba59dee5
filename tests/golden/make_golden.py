"""Generate the golden fixtures from the REAL reference package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference (`boxscreen` from
/root/reference/pkg/src), runs its `solve` on seeded inputs and stores inputs
(or the seed that regenerates them) and outputs as compressed .npz files next
to this script.  The GPU box never reads /root/reference: tests load these
fixtures instead.

Fixtures
  small_cases.npz     36 small instances (nnls/bvls/mixed x pg/cd x screening
                      on/off x 3 seeds): inputs, per-round trace, final state
  kat_cases.npz       known-answer cases from the reference test-suite shapes
  optimum_cases.npz   high-accuracy optima (active set, certified gap 1e-12)
                      for solution-level pinning of the FISTA extension
  active_cases.npz    the active-set (bounded Lawson-Hanson) solver: 18 small
                      instances (nnls/bvls/mixed x 3 seeds x screening on/off),
                      the reference suite's two KATs (test_solvers.py:144-159)
                      and a 300 x 600 screened NNLS instance
  cfg1_as_trace.npz   BASELINE config 1's instance solved by the active-set
                      kind (gap 1e-6): the reference's whole trajectory
  frontends.npz       the thin wrappers around the solver: GenSpec draws
                      (digests), estimator fits, compare_t curves,
                      solve-linear translation vectors, a CLI solve result
  cfg1_trace.npz      BASELINE config 1 at full size (1000 x 2000, PG, 10
                      passes/round, gap 1e-6): the reference's whole trajectory
  cfg2_trace.npz      BASELINE config 2 at full size (2000 x 4000, CD, gap 1e-7)
  primitives.npz      the spec-level per-round API (__init__.py exports):
                      pg_update / cd_update / active_set_update, dual points
                      (nnlr / bvlr), eval_dual, is_dual_feasible,
                      duality_gap, dual_translate, safe_screen_test,
                      apply_screening, forward_product on small instances
"""

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, REF)

import boxscreen as bs  # noqa: E402  (the reference)
import boxscreen.bench  # noqa: E402,F401

from conftest import medium_nnls, small_instance  # noqa: E402
from paper_2202_07258_b200.generate import make_config  # noqa: E402


def trace_arrays(res):
    tr = res.trace
    return dict(primal=np.array([r.primal for r in tr]), dual=np.array([r.dual for r in tr]),
                gap=np.array([r.gap for r in tr]), preserved=np.array([r.preserved_count for r in tr], np.int32),
                new_lower=np.array([r.newly_screened_lower for r in tr], np.int32),
                new_upper=np.array([r.newly_screened_upper for r in tr], np.int32))


def digest(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def small_cases():
    out = {}
    i = 0
    for family in ("nnls", "bvls", "mixed"):
        for kind in ("pg", "cd"):
            for seed in range(3):
                rng = np.random.default_rng(1000 + 17 * seed + (0 if family == "nnls" else 7 if family == "bvls" else 13))
                n = int(rng.integers(3, 31))
                m = int(rng.integers(n, 61))
                a, y, lo, hi = small_instance(rng, m, n, family)
                p = bs.Problem(a, y, lo, hi)
                for screening in (True, False):
                    res = bs.solve(p, bs.SolverConfig(kind=kind, gap_tol=1e-8, inner_passes=10),
                                   screening=screening)
                    key = f"c{i:03d}"
                    meta = np.array([family, kind, str(int(screening))])
                    out[key + "_meta"] = meta
                    out[key + "_a"] = a
                    out[key + "_y"] = y
                    out[key + "_lo"] = lo
                    out[key + "_hi"] = hi
                    for k, v in trace_arrays(res).items():
                        out[f"{key}_tr_{k}"] = v
                    out[key + "_x"] = res.x
                    out[key + "_theta"] = res.theta
                    out[key + "_final"] = np.array([res.gap, res.rounds, float(res.converged)])
                    out[key + "_sat_lower"] = np.asarray(res.sat_lower, np.int64)
                    out[key + "_sat_upper"] = np.asarray(res.sat_upper, np.int64)
                    i += 1
    out["count"] = np.array(i)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **out)
    print("small_cases:", i)


def kat_cases():
    """Known answers on the reference suite's tiny shapes, recomputed by the reference."""
    cases = [
        ("nnls1d_immediate", [[1.0]], [-1.0], 0.0, np.inf, "cd", 1),   # test_driver.py:15-22
        ("box1d_step1", [[1.0]], [3.0], 0.0, 1.0, "pg", 1),            # test_solvers.py:78-83
        ("nnls1d_cd", [[1.0]], [2.0], 0.0, np.inf, "cd", 1),           # test_solvers.py:108-113
        ("identity_nnls", np.eye(2), [1.0, -1.0], 0.0, np.inf, "pg", 10),
        ("identity_box", np.eye(2), [0.5, 0.5], -1.0, 1.0, "pg", 1),    # test_solvers.py:70-76
    ]
    out = {}
    for name, a, y, lo, hi, kind, passes in cases:
        a = np.asarray(a, float)
        n = a.shape[1]
        p = bs.Problem(a, y, lo, hi)
        step = 1.0 if name == "box1d_step1" else None
        res = bs.solve(p, bs.SolverConfig(kind=kind, inner_passes=passes, step_size=step, gap_tol=1e-6),
                       screening=True)
        out[name + "_a"] = a
        out[name + "_y"] = np.asarray(y, float)
        out[name + "_lo"] = np.broadcast_to(np.asarray(lo, float), (n,)).copy()
        out[name + "_hi"] = np.broadcast_to(np.asarray(hi, float), (n,)).copy()
        out[name + "_kind"] = np.array(kind)
        out[name + "_passes"] = np.array(passes)
        out[name + "_step"] = np.array(np.nan if step is None else step)
        out[name + "_x"] = res.x
        out[name + "_final"] = np.array([res.gap, res.rounds, float(res.converged)])
        out[name + "_ratio"] = np.array(res.trace[-1].screening_ratio)
    out["names"] = np.array([c[0] for c in cases])
    np.savez_compressed(os.path.join(HERE, "kat_cases.npz"), **out)
    print("kat_cases:", len(cases))


def optimum_cases():
    out = {}
    names = []
    for i in range(6):
        rng = np.random.default_rng(500 + i)
        fam = ("nnls", "mixed", "bvls")[i % 3]
        n = int(rng.integers(5, 25))
        m = int(rng.integers(n + 5, 60))
        a, y, lo, hi = small_instance(rng, m, n, fam)
        p = bs.Problem(a, y, lo, hi)
        res = bs.solve(p, bs.SolverConfig(kind="active-set", gap_tol=1e-12), screening=False)
        assert res.converged
        key = f"o{i}"
        names.append(key)
        out[key + "_a"] = a
        out[key + "_y"] = y
        out[key + "_lo"] = lo
        out[key + "_hi"] = hi
        out[key + "_x"] = res.x
        r = a @ res.x - y
        out[key + "_obj"] = np.array(0.5 * float(r @ r))
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "optimum_cases.npz"), **out)
    print("optimum_cases:", len(names))


def _store_case(out, key, meta, a, y, lo, hi, res):
    out[key + "_meta"] = np.array(meta)
    out[key + "_a"] = np.asarray(a, float)
    out[key + "_y"] = np.asarray(y, float)
    out[key + "_lo"] = lo
    out[key + "_hi"] = hi
    for k, v in trace_arrays(res).items():
        out[f"{key}_tr_{k}"] = v
    out[key + "_x"] = res.x
    out[key + "_theta"] = res.theta
    out[key + "_final"] = np.array([res.gap, res.rounds, float(res.converged)])
    out[key + "_sat_lower"] = np.asarray(res.sat_lower, np.int64)
    out[key + "_sat_upper"] = np.asarray(res.sat_upper, np.int64)


def active_cases():
    out = {}
    i = 0
    for family in ("nnls", "bvls", "mixed"):
        for seed in range(3):
            rng = np.random.default_rng(3000 + 31 * seed + len(family))
            n = int(rng.integers(3, 41))
            m = int(rng.integers(n, 81))
            a, y, lo, hi = small_instance(rng, m, n, family)
            for screening in (True, False):
                res = bs.solve(bs.Problem(a, y, lo, hi), bs.SolverConfig(kind="active-set", gap_tol=1e-8),
                               screening=screening)
                _store_case(out, f"c{i:03d}", [family, "active-set", str(int(screening))], a, y, lo, hi, res)
                i += 1
    # test_solvers.py:144-159 shapes
    for a, y in ((np.eye(2), [1.0, -1.0]), (np.eye(2), [-1.0, -2.0])):
        lo, hi = np.zeros(2), np.full(2, np.inf)
        res = bs.solve(bs.Problem(a, y, 0.0, np.inf), bs.SolverConfig(kind="active-set"), screening=False)
        _store_case(out, f"c{i:03d}", ["kat", "active-set", "0"], a, y, lo, hi, res)
        i += 1
    # a screened NNLS instance with a few hundred passive columns
    # (the matrix is regenerated from its seed by tests/conftest.py:medium_nnls)
    a, y, lo, hi = medium_nnls()
    res = bs.solve(bs.Problem(a, y, lo, hi), bs.SolverConfig(kind="active-set", gap_tol=1e-8), screening=True)
    key = f"c{i:03d}"
    _store_case(out, key, ["medium", "active-set", "1"], a, y, lo, hi, res)
    out[key + "_a"] = np.zeros((0, 0))
    out[key + "_digest"] = np.array(digest(a, y))
    i += 1
    out["count"] = np.array(i)
    np.savez_compressed(os.path.join(HERE, "active_cases.npz"), **out)
    print("active_cases:", i)


def frontends():
    import json
    import subprocess
    import tempfile
    out = {}
    specs = [dict(family="nnls", m=30, n=20, seed=0), dict(family="bvls", m=25, n=10, box_halfwidth=0.4, seed=1),
             dict(family="nnls", m=30, n=20, seed=2), dict(family="nnls", m=20, n=20, seed=3),
             dict(family="nnls", m=30, n=40, seed=2), dict(family="nnls", m=50, n=80, sparsity=0.1,
                                                            noise_std=0.5, seed=7)]
    out["gen_specs"] = np.array([json.dumps(sp) for sp in specs])
    out["gen_digest"] = np.array([digest(*(lambda p: (p.a_matrix, p.y, p.lower, p.upper))(
        bs.generate(bs.GenSpec(**sp)))) for sp in specs])
    out["gen_instance_hash"] = np.array([bs.bench.instance_hash(bs.generate(bs.GenSpec(**sp))) for sp in specs])
    # estimator fits (test_estimator.py shapes)
    fits = [("nnls0", specs[0], {}), ("bvls1", specs[1], dict(lower=-0.4, upper=0.4, solver="pg")),
            ("nnls2_tight", specs[2], dict(tol=1e-8)), ("nnls2_off", specs[2], dict(tol=1e-8, screening=False)),
            ("nnls3_as", specs[3], dict(solver="active-set"))]
    out["fit_names"] = np.array([f[0] for f in fits])
    for name, sp, kw in fits:
        p = bs.generate(bs.GenSpec(**sp))
        est = bs.BoxConstrainedRegression(**kw).fit(p.a_matrix, p.y)
        out[f"fit_{name}_kw"] = np.array(json.dumps(kw))
        out[f"fit_{name}_spec"] = np.array(json.dumps(sp))
        out[f"fit_{name}_coef"] = est.coef_
        out[f"fit_{name}_stats"] = np.array([est.gap_, est.n_iter_, float(est.converged_)])
    # compare_t (test_harness.py:221-229 shape)
    p = bs.generate(bs.GenSpec(**specs[4]))
    rounds, curves = bs.bench.compare_t(p, ["neg-ones", "neg-mean-column", ("neg-column", {"column": 0})])
    out["ct_labels"] = np.array(list(curves))
    out["ct_curves"] = np.array([curves[k] for k in curves])
    # solve-linear t on full-rank Gaussian columns
    rng = np.random.default_rng(77)
    a = rng.standard_normal((40, 10))
    pl = bs.Problem(a, rng.standard_normal(40), np.zeros(10), np.full(10, np.inf))
    out["sl_a"] = a
    out["sl_y"] = pl.y
    out["sl_t"] = bs.select_translation_vector(pl, "solve-linear").t
    # CLI solve on a generated instance
    with tempfile.TemporaryDirectory() as d:
        env = dict(os.environ, PYTHONPATH=REF)
        subprocess.run([sys.executable, "-m", "boxscreen.cli", "gen", "--family", "nnls", "--m", "40", "--n", "60",
                        "--seed", "5", "--out-prefix", os.path.join(d, "p")], check=True, env=env)
        subprocess.run([sys.executable, "-m", "boxscreen.cli", "solve", "--a", os.path.join(d, "p_A.mtx"), "--y",
                        os.path.join(d, "p_y.csv"), "--solver", "pg", "--inner-passes", "5", "--tol", "1e-8",
                        "--result-out", os.path.join(d, "r.json"), "--trace-out", os.path.join(d, "t.csv")],
                       check=True, env=env)
        with open(os.path.join(d, "r.json")) as fh:
            r = json.load(fh)
        out["cli_x"] = np.array(r["x"])
        out["cli_stats"] = np.array([r["gap"], r["rounds"], float(r["converged"])])
        with open(os.path.join(d, "t.csv")) as fh:
            out["cli_trace_header"] = np.array(fh.readline().strip())
    np.savez_compressed(os.path.join(HERE, "frontends.npz"), **out)
    print("frontends: ok")


def full_config(cfg_id, fname, kind=None, gap_tol=None):
    inst = make_config(cfg_id)
    p = bs.Problem(inst.a, inst.y, inst.lower, inst.upper)
    t0 = time.time()
    res = bs.solve(p, bs.SolverConfig(kind=kind or inst.kind, inner_passes=inst.inner_passes,
                                      gap_tol=gap_tol or inst.gap_tol), screening=True)
    el = time.time() - t0
    out = {f"tr_{k}": v for k, v in trace_arrays(res).items()}
    out.update(x=res.x, theta=res.theta, final=np.array([res.gap, res.rounds, float(res.converged)]),
               sat_lower=np.asarray(res.sat_lower, np.int64), sat_upper=np.asarray(res.sat_upper, np.int64),
               input_sha256=np.array(digest(inst.a, inst.y)), elapsed=np.array(el),
               step=np.array(bs.auto_step_size(inst.a, 1.0)))
    np.savez_compressed(os.path.join(HERE, fname), **out)
    print(fname, "rounds", res.rounds, "converged", res.converged, "elapsed %.1fs" % el)


def primitives():
    """One scripted sequence of the reference's per-round primitives per
    (family, seed): every input and output stored."""
    out = {}
    for fam in ("nnls", "bvls", "mixed"):
        for seed in range(2):
            rng = np.random.default_rng(1000 + seed + 10 * ("nnls", "bvls", "mixed").index(fam))
            a, y, lo, hi = small_instance(rng, 60, 40, fam)
            key = f"{fam}_{seed}"
            p = bs.Problem(a, y, lo, hi)
            st = bs.ScreeningState(p)
            pt = bs.PrimalPoint(np.clip(np.zeros(p.n), lo, hi))
            cfg = bs.SolverConfig(kind="pg", inner_passes=3000)
            step = bs.auto_step_size(a, 1.0)
            r1, g1 = bs.pg_update(p, st, pt, cfg, step)
            rec = dict(a=a, y=y, lo=lo, hi=hi, step=np.array(step), pg_r=r1, pg_g=g1, pg_x=pt.x.copy())
            tv = None
            if p.j_inf.size:
                tv = bs.select_translation_vector(p, "neg-ones")
                ds = bs.dual_point_nnlr(p, tv, pt)
                rec["t"] = tv.t
            else:
                ds = bs.dual_point_bvlr(p, pt)
            rec.update(theta=ds.theta, d_value=np.array(ds.d_value), gap=np.array(ds.gap),
                       a_t_theta=ds.a_t_theta_cache)
            rec["eval_dual"] = np.array(bs.eval_dual(p, ds.theta))
            rec["eval_dual_cached"] = np.array(bs.eval_dual(p, ds.theta, ds.a_t_theta_cache))
            rec["feasible"] = np.array(bs.is_dual_feasible(p, ds.theta))
            rec["feasible_neg"] = np.array(bs.is_dual_feasible(p, -ds.theta))
            rec["duality_gap"] = np.array(bs.duality_gap(p, pt, ds.theta))
            zg = y - a @ pt.x
            rec["zgrad"] = zg
            if tv is not None:
                rec["translated"] = bs.dual_translate(p, tv, zg)
            st.radius = bs.gap_safe_radius(ds.gap, 1.0)
            slack = 1e-12 * max(1.0, float(np.linalg.norm(ds.theta)))
            nl, nu = bs.safe_screen_test(st, ds.a_t_theta_cache, p, slack=slack)
            rec.update(radius=np.array(st.radius), slack=np.array(slack), new_lower=nl, new_upper=nu)
            # a synthetic test vector with decisions on both sides of the sphere
            vt = np.random.default_rng(seed).standard_normal(p.n) * st.col_norms
            st.radius = 0.5
            nl2, nu2 = bs.safe_screen_test(st, vt, p, slack=0.25)
            rec.update(vtest=vt, new_lower2=nl2, new_upper2=nu2)
            bs.apply_screening(st, nl, nu, pt, p)
            rec.update(z=st.z.copy(), preserved=st.preserved.copy(), x_screened=pt.x.copy())
            rec["forward"] = bs.forward_product(st, p, pt.x[st.preserved])
            r2, g2 = bs.cd_update(p, st, pt, bs.SolverConfig(kind="cd", inner_passes=3))
            rec.update(cd_r=r2, cd_g=g2, cd_x=pt.x.copy())
            # three active-set iterations from the reference's start (x = l)
            st3 = bs.ScreeningState(p)
            pt3 = bs.PrimalPoint(lo.copy())
            ass = bs.ActiveSetState(p.n)
            for it in range(3):
                r3, g3, opt = bs.active_set_update(p, st3, pt3, ass, bs.SolverConfig(kind="active-set"))
                rec.update({f"as{it}_r": r3, f"as{it}_g": g3, f"as{it}_x": pt3.x.copy(),
                            f"as{it}_passive": ass.passive.copy(), f"as{it}_opt": np.array(opt)})
            for k, v in rec.items():
                out[f"{key}/{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(HERE, "primitives.npz"), **out)
    print("primitives.npz", len(out), "arrays")


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "kat", "optimum", "active", "frontends", "cfg1as", "cfg2", "cfg1", "primitives"]
    if "primitives" in which:
        primitives()
    if "small" in which:
        small_cases()
    if "kat" in which:
        kat_cases()
    if "optimum" in which:
        optimum_cases()
    if "active" in which:
        active_cases()
    if "frontends" in which:
        frontends()
    if "cfg1as" in which:
        full_config(1, "cfg1_as_trace.npz", kind="active-set", gap_tol=1e-6)
    if "cfg2" in which:
        full_config(2, "cfg2_trace.npz")
    if "cfg1" in which:
        full_config(1, "cfg1_trace.npz")
