"""Seeded synthetic instances for the five BASELINE.json configurations.

The reference's generators (/root/reference/pkg/src/boxscreen/generate.py:39-77)
draw Gaussian/half-normal matrices; BASELINE.json asks for different recipes
(uniform or Gaussian entries with unit-norm columns, SNR-scaled noise, Gaussian
bump dictionaries), so these are new.  The stream-splitting pattern is kept:
one child ``SeedSequence`` per drawn object (generate.py:39-41), so changing a
size never perturbs the draws of the other objects.

Noise model (a documented choice, DESIGN.md section "Inputs"):
    sigma = ||A x0||_2 / sqrt(m) * 10 ** (-snr_db / 20),   y = A x0 + sigma * N(0, I_m)

Everything here is host-side numpy in fp64 (A is returned column-major).
"""

from dataclasses import dataclass

import numpy as np

PRNG_NAME = "numpy-PCG64/SeedSequence-spawn"


def _streams(seed, k):
    return [np.random.default_rng(c) for c in np.random.SeedSequence(seed).spawn(k)]


def _unit_columns(a):
    nrm = np.sqrt(np.einsum("ij,ij->j", a, a))
    a /= nrm
    return a


def _noisy(a, x0, snr_db, rng):
    clean = a @ x0
    m = a.shape[0]
    sigma = np.linalg.norm(clean) / np.sqrt(m) * 10.0 ** (-snr_db / 20.0)
    return clean + sigma * rng.standard_normal(m)


def _colmajor_uniform(rng, m, n, dtype=np.float64):
    # draw column by column order so the array is Fortran-contiguous
    return rng.random((n, m), dtype=dtype).T


@dataclass
class Instance:
    name: str
    a: np.ndarray          # (m, n), Fortran order
    y: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    x0: np.ndarray         # planted solution
    kind: str              # solver kind the config names
    inner_passes: int
    gap_tol: float


def sparse_nnls(m, n, density, snr_db, seed=0, dtype=np.float64):
    """Uniform[0,1) entries, unit columns, |N(0,1)| planted values at
    round(density*n) random positions (configs 1, 3, 4)."""
    rng_a, rng_x, rng_e = _streams(seed, 3)
    a = _unit_columns(_colmajor_uniform(rng_a, m, n, np.float64))
    k = max(1, int(round(density * n)))
    x0 = np.zeros(n)
    sup = rng_x.choice(n, size=k, replace=False)
    x0[sup] = np.abs(rng_x.standard_normal(k))
    y = _noisy(a, x0, snr_db, rng_e)
    if dtype != np.float64:
        a = np.asfortranarray(a.astype(dtype))
    return a, y, np.zeros(n), np.full(n, np.inf), x0


def sparse_nnls_block(m, n, density, snr_db, c0, c1, reduce_sum, seed=0, dtype=np.float64):
    """Columns [c0, c1) of ``sparse_nnls(m, n, ...)`` without drawing the rest:
    the A stream is advanced to column c0 (PCG64 draws one 64-bit word per
    double), so the block's columns are bit-identical to the full draw.  The
    clean signal A x0 is the sum of the ranks' partial products, formed by the
    caller's ``reduce_sum`` (an allreduce); y therefore equals the full draw's y
    up to summation order.  Returns (A_block F-order, y, lower, upper, x0)."""
    rng_a, rng_x, rng_e = _streams(seed, 3)
    rng_a.bit_generator.advance(c0 * m)
    a = _unit_columns(rng_a.random((c1 - c0, m), dtype=np.float64).T)
    k = max(1, int(round(density * n)))
    x0 = np.zeros(n)
    sup = rng_x.choice(n, size=k, replace=False)
    x0[sup] = np.abs(rng_x.standard_normal(k))
    clean = reduce_sum(a @ x0[c0:c1])
    sigma = np.linalg.norm(clean) / np.sqrt(m) * 10.0 ** (-snr_db / 20.0)
    y = clean + sigma * rng_e.standard_normal(m)
    if dtype != np.float64:
        a = np.asfortranarray(a.astype(dtype))
    return a, y, np.zeros(c1 - c0), np.full(c1 - c0, np.inf), x0


def box_bvls(m, n, snr_db, seed=0):
    """N(0,1/m) entries, unit columns, x0 40% at 0, 40% at 1, 20% U(0,1) (config 2)."""
    rng_a, rng_x, rng_e = _streams(seed, 3)
    a = np.asfortranarray(rng_a.standard_normal((n, m)).T / np.sqrt(m))
    a = _unit_columns(a)
    perm = rng_x.permutation(n)
    n0 = int(round(0.4 * n))
    n1 = int(round(0.4 * n))
    x0 = np.empty(n)
    x0[perm[:n0]] = 0.0
    x0[perm[n0:n0 + n1]] = 1.0
    rest = perm[n0 + n1:]
    x0[rest] = rng_x.random(rest.size)
    y = _noisy(a, x0, snr_db, rng_e)
    return a, y, np.zeros(n), np.ones(n), x0


def bump_dictionary(m, n, seed=0, bumps=3):
    """Columns = sum of 3 Gaussian bumps h exp(-((i-c)/w)^2/2), c~U[0,m),
    w~U[5,40) (w read as the standard deviation), h~U[0.2,1]; unit columns (config 5)."""
    (rng_a,) = _streams(seed, 1)
    i = np.arange(m, dtype=float)[:, None]
    a = np.zeros((m, n), order="F")
    for _ in range(bumps):
        c = rng_a.uniform(0.0, float(m), n)
        w = rng_a.uniform(5.0, 40.0, n)
        h = rng_a.uniform(0.2, 1.0, n)
        a += h * np.exp(-0.5 * ((i - c) / w) ** 2)
    return _unit_columns(a)


def batched_rhs(a, k_rhs, nnz=10, snr_db=30.0, seed=0):
    """K right-hand sides y_k = A x_k + noise, x_k with ``nnz`` Dirichlet(1)
    weights at random positions (config 5).  Returns (Y (m,K) F-order, X0 (n,K))."""
    rng_x, rng_e = _streams(seed + 1, 2)
    m, n = a.shape
    x0 = np.zeros((n, k_rhs), order="F")
    for k in range(k_rhs):
        sup = rng_x.choice(n, size=nnz, replace=False)
        x0[sup, k] = rng_x.dirichlet(np.ones(nnz))
    clean = a @ x0
    sig = np.linalg.norm(clean, axis=0) / np.sqrt(m) * 10.0 ** (-snr_db / 20.0)
    y = clean + sig * rng_e.standard_normal((m, k_rhs))
    return np.asfortranarray(y), x0


# BASELINE.json "configs", in order
CONFIGS = {
    1: dict(name="cfg1-nnls-pg-1000x2000-fp64", m=1000, n=2000, density=0.05, snr=30.0,
            kind="pg", inner_passes=10, gap_tol=1e-6),
    2: dict(name="cfg2-bvls-cd-2000x4000-fp64", m=2000, n=4000, snr=40.0,
            kind="cd", inner_passes=1, gap_tol=1e-7),
    3: dict(name="cfg3-nnls-apg-10000x50000-fp64", m=10000, n=50000, density=0.02, snr=30.0,
            kind="apg", inner_passes=10, gap_tol=1e-6),
    4: dict(name="cfg4-nnls-pg-20000x500000-fp32", m=20000, n=500000, density=0.005, snr=25.0,
            kind="pg", inner_passes=10, gap_tol=1e-6),
    5: dict(name="cfg5-batched-nnls-apg-200x5000xK100000-fp64", m=200, n=5000, k_rhs=100000,
            snr=30.0, kind="apg", inner_passes=10, gap_tol=1e-6),
}


def make_config(cfg_id, seed=0, m=None, n=None):
    """Build config ``cfg_id`` (1-4) at its BASELINE size, or at a scaled
    (m, n) with the same recipe when given (parity tests use small sizes)."""
    c = dict(CONFIGS[cfg_id])
    m = m or c["m"]
    n = n or c["n"]
    if cfg_id in (1, 3, 4):
        dt = np.float32 if cfg_id == 4 else np.float64
        a, y, lo, hi, x0 = sparse_nnls(m, n, c["density"], c["snr"], seed, dtype=dt)
    elif cfg_id == 2:
        a, y, lo, hi, x0 = box_bvls(m, n, c["snr"], seed)
    else:
        raise ValueError("config 5 is batched: use bump_dictionary + batched_rhs")
    return Instance(c["name"], a, y, lo, hi, x0, c["kind"], c["inner_passes"], c["gap_tol"])


# ---------------------------------------------------------------------------
# The reference's own benchmark families (generate.py:15-77): GenSpec /
# generate, used by the CLI `gen` command, the estimator tests and compare_t.
# Same streams (one spawned child per drawn object), same draws, so the same
# spec gives the same arrays as the reference (tests/test_frontends.py pins
# digests made from the reference).
# ---------------------------------------------------------------------------

@dataclass
class GenSpec:
    family: str  # "bvls" or "nnls"
    m: int
    n: int
    box_halfwidth: float = 1.0  # bvls only
    sparsity: float = 0.05      # nnls: density of the planted solution
    noise_std: float = 1.0
    seed: int = 0

    def __post_init__(self):
        from .errors import BadSpec
        if self.family not in ("bvls", "nnls"):
            raise BadSpec(f"unknown family {self.family!r}")
        if self.m < 1 or self.n < 1:
            raise BadSpec("m and n must be >= 1")
        if self.family == "bvls" and not self.box_halfwidth > 0:
            raise BadSpec("box_halfwidth must be positive")
        if self.family == "nnls":
            if not 0 < self.sparsity <= 1:
                raise BadSpec("sparsity must be in (0, 1]")
            if round(self.sparsity * self.n) < 1:
                raise BadSpec("sparsity * n must round to at least 1")


def gen_bvls(spec):
    """Gaussian box instance: A, y ~ N(0, 1) entrywise, box [-b, b]."""
    from .errors import BadSpec
    from .model import Problem
    if spec.family != "bvls":
        raise BadSpec("gen_bvls needs a bvls spec")
    s_a, s_y = _streams(spec.seed, 2)
    a = s_a.standard_normal((spec.m, spec.n))
    y = s_y.standard_normal(spec.m)
    half = spec.box_halfwidth
    return Problem(a, y, np.full(spec.n, -half), np.full(spec.n, half))


def gen_nnls(spec):
    """Half-normal matrix, planted sparse half-normal x, Gaussian noise."""
    from .errors import BadSpec, ZeroColumn
    from .model import Problem
    if spec.family != "nnls":
        raise BadSpec("gen_nnls needs an nnls spec")
    s_a, s_x, s_e = _streams(spec.seed, 3)
    a = np.abs(s_a.standard_normal((spec.m, spec.n)))
    if not np.all(np.linalg.norm(a, axis=0) > 0.0):
        raise ZeroColumn("generated matrix has a zero column")
    nnz = int(round(spec.sparsity * spec.n))
    x_true = np.zeros(spec.n)
    where = s_x.choice(spec.n, size=nnz, replace=False)
    x_true[where] = np.abs(s_x.standard_normal(nnz))
    y = a @ x_true + spec.noise_std * s_e.standard_normal(spec.m)
    return Problem(a, y, np.zeros(spec.n), np.full(spec.n, np.inf))


def generate(spec):
    return gen_nnls(spec) if spec.family == "nnls" else gen_bvls(spec)
