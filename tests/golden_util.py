"""Loaders for the reference-generated fixtures in tests/golden/ (see make_golden.py)."""
import os

import numpy as np

from oracle.oracle import Csr, Prepared

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

_cache = {}


def load(name):
    if name not in _cache:
        _cache[name] = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    return _cache[name]


def csr(d, prefix):
    dims = d[prefix + "dims"]
    return Csr(int(dims[0]), int(dims[1]), d[prefix + "rp"], d[prefix + "ci"], d[prefix + "v"])


def prepared(d, prefix):
    m = d[prefix + "meta"]
    return Prepared(int(m[0]), int(m[1]), int(m[2]), int(m[3]), d[prefix + "level_of"], d[prefix + "perm"],
                    d[prefix + "inv_perm"], d[prefix + "level_starts"], int(m[4]), d[prefix + "ell_cols"],
                    d[prefix + "ell_vals"], d[prefix + "csr_rp"], d[prefix + "csr_ci"], d[prefix + "csr_v"])


PREP_FIELDS = ["level_of", "perm", "inv_perm", "level_starts", "ell_cols", "ell_vals", "csr_rp", "csr_ci", "csr_v"]


def product_prepared_arrays(p):
    """Same field order as PREP_FIELDS, from the product's PreparedTriangular."""
    s, e = p.schedule, p.hec
    return [s.level_of, s.perm, s.inv_perm, s.level_starts, e.ell.col_indices, e.ell.values, e.csr_row_offsets,
            e.csr_col_indices, e.csr_values]


def oracle_prepared_arrays(p):
    return [p.level_of, p.perm, p.inv_perm, p.level_starts, p.ell_cols, p.ell_vals, p.csr_rp, p.csr_ci, p.csr_v]
