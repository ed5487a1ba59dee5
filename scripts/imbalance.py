"""Per-rank screening imbalance of the column-sharded configs (3 and 4).

Runs the single-GPU screened solve, reconstructs the round at which every
column left the preserved set (sat_lower / sat_upper are appended per event
in screening order, the trace gives the per-round counts), and evaluates,
for N = 2 / 4 / 8 ranks and three column assignments (contiguous blocks --
distributed.column_blocks --, strided j mod N, seeded random), the per-round
maximum and mean of the per-rank preserved counts.  A sharded step streams
each rank's preserved columns, so with the exchange cost set aside the
step time follows the busiest rank: implied efficiency
    E = sum_rounds mean_r k_r(t) / sum_rounds max_r k_r(t).

    python scripts/imbalance.py [--config 3|4] [--rounds R]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def screening_rounds(res, n):
    """round (1-based) at which each column was screened; inf = never."""
    tr = res.info["trace_arrays"]
    when = np.full(n, np.inf)
    lo_cnt = np.cumsum(tr["newly_screened_lower"])
    up_cnt = np.cumsum(tr["newly_screened_upper"])
    for arr, cum in ((res.sat_lower, lo_cnt), (res.sat_upper, up_cnt)):
        if arr.size:
            rnd = np.searchsorted(cum, np.arange(arr.size), side="right") + 1
            when[np.asarray(arr, dtype=np.int64)] = rnd
    return when


def assignment(kind, n, N):
    if kind == "contiguous":
        from paper_2202_07258_b200.distributed import column_blocks
        owner = np.empty(n, dtype=np.int64)
        for r, (c0, c1) in enumerate(column_blocks(n, N)):
            owner[c0:c1] = r
        return owner
    if kind == "strided":
        return np.arange(n) % N
    perm = np.random.default_rng(0).permutation(n)
    owner = np.empty(n, dtype=np.int64)
    owner[perm] = np.arange(n) % N
    return owner


def table(when, rounds, N_list=(2, 4, 8)):
    out = []
    n = when.size
    t = np.arange(1, rounds + 1)
    for N in N_list:
        for kind in ("contiguous", "strided", "random"):
            owner = assignment(kind, n, N)
            # preserved during round t: screened at a round >= t (or never)
            k = np.stack([np.searchsorted(np.sort(when[owner == r]), t, side="left") for r in range(N)])
            counts = np.stack([(owner == r).sum() - k[r] for r in range(N)])  # [N][rounds]
            mx, mean = counts.max(axis=0), counts.mean(axis=0)
            eff = float(mean.sum() / mx.sum())
            tail = rounds // 2
            out.append(dict(N=N, assignment=kind, efficiency=eff,
                            max_over_mean_worst=float((mx / np.maximum(mean, 1e-9)).max()),
                            max_over_mean_tail=float(mx[tail:].sum() / mean[tail:].sum()),
                            final_counts=[int(c) for c in counts[:, -1]]))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=100, help="config 4: screened rounds")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import bench
    from paper_2202_07258_b200 import Problem, SolverConfig, solve
    inst = bench.make_instance(args.config)
    p = Problem(inst.a, inst.y, inst.lower, inst.upper, dtype=inst.a.dtype)
    cfg = SolverConfig(kind=inst.kind, inner_passes=inst.inner_passes, gap_tol=inst.gap_tol,
                       max_rounds=args.rounds if args.config == 4 else None)
    res = solve(p, cfg)
    n = inst.a.shape[1]
    when = screening_rounds(res, n)
    assert int(np.isfinite(when).sum()) == res.sat_lower.size + res.sat_upper.size
    rows = table(when, res.rounds)
    doc = dict(config=args.config, n=n, rounds=res.rounds, screened=int(np.isfinite(when).sum()),
               final_preserved=int(res.trace[-1].preserved_count), rows=rows)
    text = json.dumps(doc, indent=1)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text)
    for r in rows:
        print(f"N={r['N']} {r['assignment']:>10}: efficiency {r['efficiency']:.4f}  "
              f"max/mean tail {r['max_over_mean_tail']:.4f} worst {r['max_over_mean_worst']:.3f}  "
              f"final per-rank {r['final_counts']}")


if __name__ == "__main__":
    main()
