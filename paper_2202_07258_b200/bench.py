"""The reference's benchmark protocols over the GPU solver.

Contract kept from /root/reference/pkg/src/boxscreen/bench.py (the API and
the files a user's scripts read): ``BenchRow`` / ``BenchReport`` with the
same fields, ``run_bench(specs, solvers, repetitions, gap_tol)`` (paired
screening off / on, median of the repetitions, speedup = off / on, failing
cells reported under ``meta["errors"]``, ``BOXSCREEN_THREADS`` host
threads), ``compare_t`` (screening-ratio curves per translation strategy on
a common round grid), the CSV column schemas and the JSON layout.

How it runs here: each cell uploads its generated problem to the device once
(every solve of the cell reuses those buffers), and timings are the native
loop's ``trace[-1].elapsed`` -- with screening off the device time of the
gap evaluation is subtracted, the reference's offline-gap convention
(driver.py:180-181).  Not the repo's headline bench (``/bench.py`` measures
the BASELINE configs).
"""

import csv
import hashlib
import json
import os
import statistics
from concurrent.futures import ThreadPoolExecutor
from dataclasses import asdict, dataclass, field

import numpy as np

from .driver import solve
from .duality import select_translation_vector
from .generate import PRNG_NAME, generate
from .solvers import SolverConfig

THREADS_ENV = "BOXSCREEN_THREADS"


def instance_hash(p):
    """16 hex digits of sha256(A, y, lower, upper) -- bench.py:19-25's
    instance identity, from the host copy (or the device copy of a
    device-built problem)."""
    if p.a_matrix is not None:
        parts = (p.a_matrix, p.y)
    else:
        dev = p.device_arrays()
        parts = (dev["a"][:, : p.m].double().T.cpu().numpy(), dev["y"].cpu().numpy())
    digest = hashlib.sha256()
    for arr in parts + (p.lower, p.upper):
        digest.update(np.asarray(arr).tobytes())
    return digest.hexdigest()[:16]


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


# CSV schemas of the reference's reports: (header, value of a record)
_ROW_SCHEMA = (
    ("solver", lambda r: r.solver),
    ("screening", lambda r: "on" if r.screening else "off"),
    ("family", lambda r: r.family), ("m", lambda r: r.m), ("n", lambda r: r.n), ("seed", lambda r: r.seed),
    ("elapsed_s", lambda r: format(r.elapsed, ".9f")),
    ("rounds", lambda r: r.rounds),
    ("gap", lambda r: format(r.gap, ".17g")),
    ("ratio", lambda r: format(r.screening_ratio, ".17g")),
    ("instance", lambda r: r.instance),
)
_SPEEDUP_SCHEMA = (
    ("solver", lambda s: s["solver"]), ("family", lambda s: s["family"]), ("m", lambda s: s["m"]),
    ("n", lambda s: s["n"]), ("seed", lambda s: s["seed"]),
    ("elapsed_off_s", lambda s: format(s["elapsed_off"], ".9f")),
    ("elapsed_on_s", lambda s: format(s["elapsed_on"], ".9f")),
    ("speedup", lambda s: format(s["speedup"], ".6g")),
    ("ratio_on", lambda s: format(s["ratio_on"], ".17g")),
)


def _write_table(path, schema, records):
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow([name for name, _ in schema])
        out.writerows([[get(rec) for _, get in schema] for rec in records])


@dataclass
class BenchReport:
    rows: list = field(default_factory=list)
    speedups: list = field(default_factory=list)
    meta: dict = field(default_factory=lambda: {"prng": PRNG_NAME})

    def to_json(self, path=None, indent=2):
        payload = {"meta": self.meta, "rows": [asdict(r) for r in self.rows], "speedups": self.speedups}
        text = json.dumps(payload, indent=indent)
        if path is not None:
            with open(path, "w") as fh:
                fh.write(text)
        return text

    def rows_to_csv(self, path):
        _write_table(path, _ROW_SCHEMA, self.rows)

    def speedups_to_csv(self, path):
        _write_table(path, _SPEEDUP_SCHEMA, self.speedups)


class _Cell:
    """One (spec, solver) pair of the sweep: paired off / on timings."""

    def __init__(self, spec, solver, repetitions, gap_tol):
        self.spec, self.solver = spec, solver
        self.repetitions, self.gap_tol = repetitions, gap_tol

    def _ident(self):
        s = self.spec
        return {"solver": self.solver, "family": s.family, "m": s.m, "n": s.n, "seed": s.seed}

    def _median(self, p, tv, screening):
        cfg = SolverConfig(kind=self.solver, gap_tol=self.gap_tol)
        runs = [solve(p, cfg, screening=screening, tv=tv) for _ in range(self.repetitions)]
        return statistics.median(r.trace[-1].elapsed for r in runs), runs[-1]

    def run(self):
        """(rows, speedup dict) -- or ([], ident + error) when the cell fails."""
        try:
            p = generate(self.spec)
            p.device_arrays()  # one upload; every solve of the cell reuses it
            tv = select_translation_vector(p, "neg-ones") if p.j_inf.size else None
            key = instance_hash(p)
            timed = {flag: self._median(p, tv, flag) for flag in (False, True)}
        except Exception as exc:  # a failing cell is reported, the sweep goes on
            return [], dict(self._ident(), error=f"{type(exc).__name__}: {exc}")
        s = self.spec
        rows = [BenchRow(self.solver, flag, s.family, s.m, s.n, s.seed, t, r.rounds, r.gap,
                         r.trace[-1].screening_ratio, key) for flag, (t, r) in timed.items()]
        (t_off, _), (t_on, r_on) = timed[False], timed[True]
        speedup = dict(self._ident(), elapsed_off=t_off, elapsed_on=t_on, speedup=t_off / t_on,
                       ratio_on=r_on.trace[-1].screening_ratio, instance=key)
        return rows, speedup


def run_bench(specs, solvers, repetitions=5, gap_tol=1e-6):
    """Paired screening-off / screening-on sweep over (spec, solver) cells."""
    if repetitions < 1:
        raise ValueError("repetitions must be >= 1")
    cells = [_Cell(spec, solver, repetitions, gap_tol) for spec in specs for solver in solvers]
    workers = int(os.environ.get(THREADS_ENV, "1"))
    if workers > 1:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            outcomes = list(pool.map(_Cell.run, cells))
    else:
        outcomes = [cell.run() for cell in cells]
    report = BenchReport()
    report.meta.update(repetitions=repetitions, gap_tol=gap_tol)
    for rows, speedup in outcomes:
        report.rows += rows
        (report.meta.setdefault("errors", []) if "error" in speedup else report.speedups).append(speedup)
    return report


def compare_t(p, strategies, solver="cd", gap_tol=1e-6, columns=None):
    """Screening ratio per round for each translation strategy, padded with
    each curve's final value to the longest run.  Returns (rounds, {label:
    ratios})."""
    curves = {}
    for entry in strategies:
        name, kwargs = entry if isinstance(entry, tuple) else (entry, {})
        res = solve(p, SolverConfig(kind=solver, gap_tol=gap_tol), screening=True,
                    tv=select_translation_vector(p, name, **kwargs))
        curves[f"{name}:{kwargs.get('column')}" if kwargs else name] = [t.screening_ratio for t in res.trace]
    span = max(map(len, curves.values()))
    padded = {label: c + [c[-1]] * (span - len(c)) for label, c in curves.items()}
    return list(range(1, span + 1)), padded


def compare_t_to_csv(rounds, curves, path):
    labels = list(curves)
    _write_table(path, [("round", lambda i: rounds[i])] +
                 [(lab, (lambda lab_: lambda i: format(curves[lab_][i], ".17g"))(lab)) for lab in labels],
                 range(len(rounds)))
