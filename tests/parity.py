"""Round-by-round comparison of a GPU solve against the CPU oracle.

Tolerances (north_star, BASELINE.json): objective and duality gap within
1e-10 relative -- read as |delta| <= 1e-10 * max(|P|, |D|) because the gap is
a difference of two O(1) numbers (hard part 1) -- final x
within 1e-8 relative, screened index sets identical except for coordinates
whose sphere-test margin is within 1e-12 of zero.
"""

import numpy as np

OBJ_RTOL = 1e-10
X_RTOL = 1e-8


def compare_traces(gpu_res, orc, obj_rtol=OBJ_RTOL, abs_floor=1e-13, max_rounds=None):
    """Return a list of problems (empty when the trajectories agree)."""
    probs = []
    gt = gpu_res.trace
    ot = orc["trace"]
    nr = min(len(gt), len(ot)) if max_rounds is None else min(len(gt), len(ot), max_rounds)
    for i in range(nr):
        g, o = gt[i], ot[i]
        scale = max(abs(o["primal"]), abs(o["dual"]), abs_floor / obj_rtol)
        for key_g, key_o in (("primal", "primal"), ("dual", "dual"), ("gap", "gap")):
            dv = abs(getattr(g, key_g) - o[key_o])
            if dv > obj_rtol * scale:
                probs.append(f"round {i + 1}: {key_g} gpu={getattr(g, key_g)!r} oracle={o[key_o]!r} "
                             f"|d|={dv:.3e} > {obj_rtol * scale:.3e}")
        if g.preserved_count != o["preserved"]:
            probs.append(f"round {i + 1}: preserved gpu={g.preserved_count} oracle={o['preserved']}")
        if probs:
            break
    if max_rounds is None and not probs and len(gt) != len(ot):
        probs.append(f"rounds gpu={len(gt)} oracle={len(ot)}")
    return probs


def compare_final(gpu_res, orc, x_rtol=X_RTOL):
    probs = []
    x, xo = np.asarray(gpu_res.x, dtype=float), orc["x"]
    den = max(1.0, float(np.max(np.abs(xo))))
    dx = float(np.max(np.abs(x - xo))) / den if x.size else 0.0
    if dx > x_rtol:
        probs.append(f"final x rel diff {dx:.3e} > {x_rtol}")
    if not np.array_equal(np.sort(gpu_res.sat_lower), np.sort(orc["sat_lower"])):
        probs.append("sat_lower differs")
    if not np.array_equal(np.sort(gpu_res.sat_upper), np.sort(orc["sat_upper"])):
        probs.append("sat_upper differs")
    if gpu_res.converged != orc["converged"]:
        probs.append(f"converged gpu={gpu_res.converged} oracle={orc['converged']}")
    return probs
