"""Column-sharded restatement of the oracle's PG / FISTA round (test
infrastructure).  It follows the data flow of the native sharded loop
(csrc/bx_core.cu: run_reduce phase A/B, dual_point, k_scan global counts): the
only cross-rank quantities are the partial A x rows (SUM), the dual-translation
epsilon (MAX), the dual bound terms (SUM) and the screening counts (SUM).
``allreduce(array, op)`` is supplied by the caller (torch.distributed gloo in
tests/test_distributed_cpu.py)."""

import math

import numpy as np


def sharded_rounds(a, y, lo, hi, col_offset, n_global, kind, eta, rounds, passes, allreduce,
                   slack_scale=1e-12, t=None):
    m = a.shape[0]
    t = -np.ones(m) if t is None else t
    inf_local = np.isinf(hi)
    has_inf = allreduce(np.array([float(inf_local.any())]), "max")[0] > 0
    norms = np.linalg.norm(a, axis=0)
    att = a.T @ t
    keep = np.arange(a.shape[1])
    x = np.clip(np.zeros(a.shape[1]), lo, hi)
    z = np.zeros(m)

    def resid(xk, kp):
        return allreduce(a[:, kp] @ xk, "sum") + (z - y)

    r = resid(x[keep], keep)
    g_cur = a[:, keep].T @ r            # this rank's columns of A'r (r is replicated)
    x_prev, g_prev, mom = x.copy(), g_cur.copy(), 1.0
    out = []
    for _ in range(rounds):
        xa = x[keep]
        obj = 0.5 * float(r @ r)
        for _ in range(passes):
            if kind == "pg":
                g = allreduce(np.zeros(0), "sum") if False else a[:, keep].T @ r
                xn = np.clip(xa - eta * g, lo[keep], hi[keep])
                r = resid(xn, keep)
                xa = xn
            else:
                tn = (1.0 + math.sqrt(1.0 + 4.0 * mom * mom)) / 2.0
                beta = (mom - 1.0) / tn
                xp = x_prev[keep]
                yv = xa + beta * (xa - xp) if beta != 0.0 else xa
                gy = g_cur + beta * (g_cur - g_prev) if beta != 0.0 else g_cur
                xn = np.clip(yv - eta * gy, lo[keep], hi[keep])
                rn = resid(xn, keep)
                nobj = 0.5 * float(rn @ rn)
                dx = xn - xa
                gd = allreduce(np.array([float(gy @ dx), float(norms[keep] @ np.abs(dx))]), "sum")
                s_f = 1e-12 * max(1.0, abs(obj))
                s_g = 1e-12 * math.sqrt(2.0 * obj) * gd[1]
                x_prev[keep] = xa
                g_prev = g_cur
                mom = 1.0 if (nobj > obj + s_f or gd[0] > s_g) else tn
                xa, r, obj = xn, rn, nobj
                g_cur = a[:, keep].T @ r
        x[keep] = xa
        g = a[:, keep].T @ r
        v = -g
        eps = 0.0
        if has_inf:
            here = inf_local[keep]
            loc = float(np.max(np.maximum(v[here], 0.0) / np.abs(att[keep][here]))) if here.any() else 0.0
            eps = allreduce(np.array([loc]), "max")[0]
            v = v + eps * att[keep]
        theta = -r + eps * t if eps > 0.0 else -r
        primal = 0.5 * float(r @ r)
        fin = ~np.isinf(hi[keep])
        bnd = allreduce(np.array([float(lo[keep] @ np.minimum(v, 0.0)),
                                  float(hi[keep][fin] @ np.maximum(v[fin], 0.0)) if fin.any() else 0.0]), "sum")
        dual = float(theta @ (y - z)) - 0.5 * float(theta @ theta) - bnd[0] - bnd[1]
        gap = max(primal - dual, 0.0)
        radius = math.sqrt(2.0 * gap)
        slack = slack_scale * max(1.0, float(np.linalg.norm(theta)))
        thr = (radius + slack) * norms[keep]
        new_lo = keep[v < -thr]
        new_up = keep[(v > thr) & fin]
        cnt = allreduce(np.array([float(new_lo.size), float(new_up.size)]), "sum")
        if cnt.sum() > 0:
            x[new_lo] = lo[new_lo]
            x[new_up] = hi[new_up]
            zc = a[:, new_lo] @ lo[new_lo] + a[:, new_up] @ hi[new_up]
            z = z + allreduce(zc, "sum")
            gone = np.concatenate([new_lo, new_up])
            x_prev[gone] = x[gone]
            keep = keep[~np.isin(keep, gone)]
            r = resid(x[keep], keep)
            g_cur = a[:, keep].T @ r
            g_prev = a[:, keep].T @ resid(x_prev[keep], keep)
        kg = allreduce(np.array([float(keep.size)]), "sum")[0]
        out.append(dict(primal=primal, dual=dual, gap=gap, preserved=int(kg)))
    return out, x
