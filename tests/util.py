"""Shared test helpers: seeded numpy generators shaped like the reference's
test_helpers.hpp (random_lower / random_upper / random_diag_dominant: the
diagonal is sum|offdiag| + 1), conversion between the product's CsrMatrix and
the oracle's Csr, and bitwise comparison."""
import numpy as np

from oracle.oracle import Csr

I32, F64 = np.int32, np.float64


def bits_equal(a, b) -> bool:
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    return a.size == 0 or bool((a.view(np.uint8) == b.view(np.uint8)).all())


def rel_inf_error(got, want) -> float:
    den = np.max(np.abs(want)) if len(want) else 0.0
    num = np.max(np.abs(np.asarray(got) - np.asarray(want))) if len(want) else 0.0
    return num / den if den > 0 else num


def _csr_from_rows(n, rows):
    rp = np.zeros(n + 1, I32)
    ci, v = [], []
    for i, (cols, vals) in enumerate(rows):
        order = np.argsort(cols, kind="stable")
        ci.extend(np.asarray(cols)[order].tolist())
        v.extend(np.asarray(vals)[order].tolist())
        rp[i + 1] = len(ci)
    return Csr(n, n, rp, np.array(ci, I32), np.array(v, F64))


def random_triangular(n, density, rng, upper=False) -> Csr:
    rows = []
    for i in range(n):
        span = (n - 1 - i) if upper else i
        k = int(density * span)
        picks = rng.choice(span, size=k, replace=False) if k else np.zeros(0, int)
        cols = (i + 1 + picks) if upper else picks
        vals = rng.uniform(-1.0, 1.0, size=k)
        d = float(np.sum(np.abs(vals))) + 1.0
        rows.append((np.append(cols, i).astype(int), np.append(vals, d)))
    return _csr_from_rows(n, rows)


def random_diag_dominant(n, density, rng) -> Csr:
    rows = []
    for i in range(n):
        k = int(density * (n - 1))
        picks = rng.choice(n - 1, size=k, replace=False) if k else np.zeros(0, int)
        cols = np.where(picks >= i, picks + 1, picks)
        vals = rng.uniform(-1.0, 1.0, size=k)
        rows.append((np.append(cols, i).astype(int), np.append(vals, float(np.sum(np.abs(vals))) + 1.0)))
    return _csr_from_rows(n, rows)


def to_product(H, a: Csr):
    return H.CsrMatrix.from_arrays(a.n_rows, a.n_cols, a.rp, a.ci, a.v)


def to_oracle(m) -> Csr:
    return Csr.of(m)
