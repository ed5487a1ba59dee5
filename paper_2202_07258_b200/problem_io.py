"""Problem ingestion and serialisation (reference problem_io.py:1-122).

Formats, as in the reference: the matrix as Matrix Market (``.mtx`` /
``.mm``; array or coordinate, densified) or a headerless CSV; y as a
one-column CSV; bounds as ``nn``, ``box:lo:hi`` or a two-column CSV whose
upper column may hold ``inf``.  Malformed files raise ``ParseError`` with the
line / column, shape disagreements ``DimensionMismatch``, and all-zero
columns / rows ``ZeroColumn`` / ``ZeroRow``.

Text parsing is host work; everything after it runs on the device.  With
``device="cuda"`` (the default when a GPU is present) the parsed matrix is
uploaded once into the solver's column-major layout, the column and row norms
(zero column / row rejection) and the optional column normalisation are
computed there, and the returned ``Problem`` is device-resident -- the solve
then starts without another host copy.  ``device=None`` keeps the reference's
host ``Problem`` (fp64 numpy).
"""

import os

import numpy as np

from .errors import DimensionMismatch, ParseError, ZeroColumn, ZeroRow
from .model import Problem

FLOAT_FMT = "%.17g"
_INF_TOKENS = ("inf", "+inf", "infinity", "+infinity")


def read_csv_array(path, ncols=None):
    """Numbers of a headerless CSV as a 2-d float array (problem_io.py:34-63)."""
    rows = []
    width = None
    with open(path) as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.strip()
            if not line:
                continue
            vals = []
            for colno, tok in enumerate(line.split(","), start=1):
                tok = tok.strip()
                if tok.lower() in _INF_TOKENS:
                    vals.append(np.inf)
                    continue
                try:
                    vals.append(float(tok))
                except ValueError:
                    raise ParseError(f"{path}: line {lineno}, column {colno}: cannot parse {tok!r} as a number")
            if ncols is not None and len(vals) != ncols:
                raise ParseError(f"{path}: line {lineno}: expected {ncols} fields, got {len(vals)}")
            if width is not None and len(vals) != width:
                raise ParseError(f"{path}: line {lineno}: ragged row ({len(vals)} fields, "
                                 f"previous rows have {width})")
            width = len(vals)
            rows.append(vals)
    if not rows:
        raise ParseError(f"{path}: empty file")
    return np.asarray(rows, dtype=float)


def read_matrix(path):
    """Matrix Market (dense or coordinate, densified) or CSV."""
    if str(path).endswith((".mtx", ".mm")):
        import scipy.io
        import scipy.sparse
        try:
            a = scipy.io.mmread(path)
        except Exception as exc:
            raise ParseError(f"{path}: invalid Matrix Market file: {exc}")
        if scipy.sparse.issparse(a):
            a = a.toarray()
        return np.asarray(a, dtype=float)
    return read_csv_array(path)


def parse_bounds(spec, n):
    """'nn' | 'box:lo:hi' | path of a two-column CSV -> (lower, upper)."""
    if spec == "nn":
        return np.zeros(n), np.full(n, np.inf)
    if isinstance(spec, str) and spec.startswith("box:"):
        parts = spec.split(":")
        if len(parts) != 3:
            raise ParseError(f"bad bounds spec {spec!r}; want box:lo:hi")
        try:
            lo, hi = float(parts[1]), float(parts[2])
        except ValueError:
            raise ParseError(f"bad bounds spec {spec!r}: non-numeric limit")
        return np.full(n, lo), np.full(n, hi)
    if isinstance(spec, str) and os.path.exists(spec):
        arr = read_csv_array(spec, ncols=2)
        if arr.shape[0] != n:
            raise DimensionMismatch(f"bounds file has {arr.shape[0]} rows, expected {n}")
        return arr[:, 0].copy(), arr[:, 1].copy()
    raise ParseError(f"bad bounds spec {spec!r}; want 'nn', 'box:lo:hi' or an existing CSV path")


def _default_device():
    try:
        import torch
        return "cuda" if torch.cuda.is_available() else None
    except ImportError:  # pragma: no cover
        return None


def load_problem(path_a, path_y, bounds_spec, normalize_columns=False, device="auto", dtype=np.float64):
    """Read, validate and assemble a Problem (problem_io.py:88-108)."""
    a = read_matrix(path_a)
    if a.ndim != 2:
        raise ParseError(f"{path_a}: expected a 2-d matrix")
    y = read_csv_array(path_y, ncols=1).ravel()
    if y.shape[0] != a.shape[0]:
        raise DimensionMismatch(f"y has length {y.shape[0]}, matrix has {a.shape[0]} rows")
    if device == "auto":
        device = _default_device()
    if device is None:
        col = np.linalg.norm(a, axis=0)
        zc = np.flatnonzero(col == 0.0)
        if zc.size:
            raise ZeroColumn(f"{path_a}: all-zero column(s) {zc.tolist()}")
        zr = np.flatnonzero(np.linalg.norm(a, axis=1) == 0.0)
        if zr.size:
            raise ZeroRow(f"{path_a}: all-zero row(s) {zr.tolist()}")
        if normalize_columns:
            a = a / col
        lower, upper = parse_bounds(bounds_spec, a.shape[1])
        return Problem(a, y, lower, upper, dtype=dtype)
    import torch
    # one upload into the column-major (n, m) storage the kernels stream
    at = torch.from_numpy(np.ascontiguousarray(a.T)).to(device)
    col = torch.linalg.vector_norm(at, dim=1)
    zc = torch.nonzero(col == 0.0).ravel()
    if zc.numel():
        raise ZeroColumn(f"{path_a}: all-zero column(s) {zc.cpu().tolist()}")
    zr = torch.nonzero(torch.linalg.vector_norm(at, dim=0) == 0.0).ravel()
    if zr.numel():
        raise ZeroRow(f"{path_a}: all-zero row(s) {zr.cpu().tolist()}")
    if normalize_columns:
        at = at / col[:, None]
    lower, upper = parse_bounds(bounds_spec, a.shape[1])
    tdt = torch.float32 if np.dtype(dtype) == np.float32 else torch.float64
    return Problem(at.T.to(tdt), torch.from_numpy(y).to(device), lower, upper)


def save_problem(p, prefix):
    """Write <prefix>_A.mtx, <prefix>_y.csv and <prefix>_bounds.csv."""
    import scipy.io
    a = p.a_matrix
    y = p.y
    if a is None:  # device-resident problem
        st = p.device_arrays()["a"]
        a = st[:, : p.m].double().T.cpu().numpy()
        y = p.device_arrays()["y"].cpu().numpy()
    path_a, path_y, path_b = f"{prefix}_A.mtx", f"{prefix}_y.csv", f"{prefix}_bounds.csv"
    scipy.io.mmwrite(path_a, np.asarray(a, dtype=float))
    np.savetxt(path_y, np.asarray(y, dtype=float)[:, None], fmt=FLOAT_FMT, delimiter=",")
    with open(path_b, "w") as fh:
        for lo, hi in zip(p.lower, p.upper):
            fh.write((FLOAT_FMT % lo) + "," + ("inf" if np.isinf(hi) else FLOAT_FMT % hi) + "\n")
    return path_a, path_y, path_b
