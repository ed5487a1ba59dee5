"""Benchmark protocols of the reference (bench.py:19-184) over the GPU solver.

* ``run_bench`` -- paired screening-off / screening-on timings per
  (GenSpec, solver) cell, median of ``repetitions`` solves, speedup =
  off / on.  Timings follow the reference's offline-gap convention: with
  screening off the gap evaluation is excluded from ``trace[-1].elapsed``
  (the native loop subtracts the device time of the dual / gap kernels).
  Independent cells run on up to ``BOXSCREEN_THREADS`` host threads; a failing
  cell is recorded under ``meta["errors"]`` instead of aborting the sweep.
* ``compare_t`` -- screening-ratio-per-round curves for several translation
  vector strategies, padded to a common round grid.

This is the reference's user-facing protocol, not the repo's headline bench
(``/bench.py`` at the repository root measures the BASELINE configs).
"""

import csv
import hashlib
import json
import os
import statistics
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from .driver import solve
from .duality import select_translation_vector
from .generate import PRNG_NAME, generate
from .solvers import SolverConfig

THREADS_ENV = "BOXSCREEN_THREADS"


def _host_arrays(p):
    if p.a_matrix is not None:
        return p.a_matrix, p.y
    d = p.device_arrays()
    return d["a"][:, : p.m].double().T.cpu().numpy(), d["y"].cpu().numpy()


def instance_hash(p):
    """First 16 hex digits of sha256 over A, y, lower, upper (bench.py:19-25)."""
    a, y = _host_arrays(p)
    h = hashlib.sha256()
    for arr in (a, y, p.lower, p.upper):
        h.update(np.asarray(arr).tobytes())
    return h.hexdigest()[:16]


@dataclass
class BenchRow:
    solver: str
    screening: bool
    family: str
    m: int
    n: int
    seed: int
    elapsed: float
    rounds: int
    gap: float
    screening_ratio: float
    instance: str


@dataclass
class BenchReport:
    rows: list = field(default_factory=list)
    speedups: list = field(default_factory=list)
    meta: dict = field(default_factory=lambda: {"prng": PRNG_NAME})

    def to_json(self, path=None, indent=2):
        text = json.dumps({"meta": self.meta, "rows": [vars(r) for r in self.rows], "speedups": self.speedups},
                          indent=indent)
        if path is not None:
            with open(path, "w") as fh:
                fh.write(text)
        return text

    def rows_to_csv(self, path):
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["solver", "screening", "family", "m", "n", "seed", "elapsed_s", "rounds", "gap", "ratio",
                        "instance"])
            for r in self.rows:
                w.writerow([r.solver, "on" if r.screening else "off", r.family, r.m, r.n, r.seed,
                            f"{r.elapsed:.9f}", r.rounds, f"{r.gap:.17g}", f"{r.screening_ratio:.17g}", r.instance])

    def speedups_to_csv(self, path):
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["solver", "family", "m", "n", "seed", "elapsed_off_s", "elapsed_on_s", "speedup",
                        "ratio_on"])
            for s in self.speedups:
                w.writerow([s["solver"], s["family"], s["m"], s["n"], s["seed"], f"{s['elapsed_off']:.9f}",
                            f"{s['elapsed_on']:.9f}", f"{s['speedup']:.6g}", f"{s['ratio_on']:.17g}"])


def _median_solve(p, solver, screening, repetitions, gap_tol, tv):
    times, last = [], None
    for _ in range(repetitions):
        last = solve(p, SolverConfig(kind=solver, gap_tol=gap_tol), screening=screening, tv=tv)
        times.append(last.trace[-1].elapsed)
    return statistics.median(times), last


def _cell(spec, solver, repetitions, gap_tol):
    p = generate(spec)
    tv = select_translation_vector(p, "neg-ones") if p.j_inf.size else None
    inst = instance_hash(p)
    rows = []
    timed = {}
    for screening in (False, True):
        t, res = _median_solve(p, solver, screening, repetitions, gap_tol, tv)
        timed[screening] = (t, res)
        rows.append(BenchRow(solver, screening, spec.family, spec.m, spec.n, spec.seed, t, res.rounds, res.gap,
                             res.trace[-1].screening_ratio, inst))
    (t_off, _), (t_on, r_on) = timed[False], timed[True]
    return rows, dict(solver=solver, family=spec.family, m=spec.m, n=spec.n, seed=spec.seed, elapsed_off=t_off,
                      elapsed_on=t_on, speedup=t_off / t_on, ratio_on=r_on.trace[-1].screening_ratio,
                      instance=inst)


def run_bench(specs, solvers, repetitions=5, gap_tol=1e-6):
    """Paired off / on sweep over (spec, solver) cells (bench.py:118-152)."""
    if repetitions < 1:
        raise ValueError("repetitions must be >= 1")
    cells = [(spec, solver) for spec in specs for solver in solvers]
    report = BenchReport()
    report.meta.update(repetitions=repetitions, gap_tol=gap_tol)

    def one(cell):
        spec, solver = cell
        try:
            return _cell(spec, solver, repetitions, gap_tol)
        except Exception as exc:  # a failing cell must not abort the sweep
            return [], dict(solver=solver, family=spec.family, m=spec.m, n=spec.n, seed=spec.seed,
                            error=f"{type(exc).__name__}: {exc}")

    threads = int(os.environ.get(THREADS_ENV, "1"))
    if threads > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            results = list(pool.map(one, cells))
    else:
        results = [one(c) for c in cells]
    for rows, sp in results:
        report.rows.extend(rows)
        if "error" in sp:
            report.meta.setdefault("errors", []).append(sp)
        else:
            report.speedups.append(sp)
    return report


def compare_t(p, strategies, solver="cd", gap_tol=1e-6, columns=None):
    """Screening ratio per round for each translation strategy (bench.py:155-176).

    ``strategies`` holds names or (name, kwargs) pairs; curves are padded with
    their last ratio to the longest run.  Returns (rounds, {label: ratios}).
    """
    curves = {}
    for strat in strategies:
        name, kwargs = strat if isinstance(strat, tuple) else (strat, {})
        tv = select_translation_vector(p, name, **kwargs)
        res = solve(p, SolverConfig(kind=solver, gap_tol=gap_tol), screening=True, tv=tv)
        label = f"{name}:{kwargs.get('column')}" if kwargs else name
        curves[label] = [rec.screening_ratio for rec in res.trace]
    longest = max(len(c) for c in curves.values())
    for c in curves.values():
        c.extend([c[-1]] * (longest - len(c)))
    return list(range(1, longest + 1)), curves


def compare_t_to_csv(rounds, curves, path):
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["round"] + list(curves))
        for i, rnd in enumerate(rounds):
            w.writerow([rnd] + [f"{curves[k][i]:.17g}" for k in curves])
