"""Probe for the reference's criterion 6 (pkg/tests/test_acceptance.py:203-232)
on the GPU path: per box half-width, the saturation of the solution, the work
ratio (column updates off / on) and the device-time ratio of PG solves."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from paper_2202_07258_b200 import SolverConfig, solve  # noqa: E402
from paper_2202_07258_b200.generate import GenSpec, generate  # noqa: E402
from paper_2202_07258_b200.solvers import auto_step_size  # noqa: E402

for b in np.logspace(np.log10(0.01), np.log10(3.0), 12):
    p = generate(GenSpec("bvls", 400, 200, box_halfwidth=float(b), seed=5))
    eta = auto_step_size(p.a_matrix, 1.0)
    cfg = SolverConfig(kind="pg", inner_passes=30, step_size=eta, gap_tol=1e-9)
    t_off = min(solve(p, cfg, screening=False).trace[-1].elapsed for _ in range(5))
    ons = [solve(p, cfg, screening=True) for _ in range(5)]
    t_on = min(r.trace[-1].elapsed for r in ons)
    off = solve(p, cfg, screening=False)
    on = ons[0]
    pres = [t.preserved_count for t in on.trace]
    w_on = 200 + sum(pres[:-1])
    w_off = off.rounds * 200
    ref = solve(p, SolverConfig(kind="active-set"), screening=False)
    sat = float(np.mean((np.abs(ref.x - p.lower) < 1e-7) | (np.abs(ref.x - p.upper) < 1e-7)))
    print(f"b={b:.3f} sat={sat:.2f} rounds off/on {off.rounds}/{on.rounds} work ratio {w_off / w_on:.2f} "
          f"time ratio {t_off / t_on:.2f}", flush=True)
