"""ctypes front-ends for the two checkers (see oracle/__init__.py).

Both work on plain numpy CSR triples ``(n, rp, ci, v)`` so they never touch the
product library.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libhecoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhecref.so")

I32, F64 = np.int32, np.float64
P_int, P_dbl, P_chr = C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_char)


def _pi(a):
    return a.ctypes.data_as(P_int)


def _pd(a):
    return a.ctypes.data_as(P_dbl)


@dataclass
class Csr:
    n_rows: int
    n_cols: int
    rp: np.ndarray
    ci: np.ndarray
    v: np.ndarray

    def __post_init__(self):
        self.rp = np.ascontiguousarray(self.rp, dtype=I32)
        self.ci = np.ascontiguousarray(self.ci, dtype=I32)
        self.v = np.ascontiguousarray(self.v, dtype=F64)

    @property
    def n(self):
        return self.n_rows

    @staticmethod
    def of(m) -> "Csr":
        """From any object with the reference field names (e.g. the product's CsrMatrix)."""
        return Csr(m.n_rows, m.n_cols, np.array(m.row_offsets, dtype=I32), np.array(m.col_indices, dtype=I32),
                   np.array(m.values, dtype=F64))


@dataclass
class Prepared:
    kind: int
    n: int
    reversed: int
    nlev: int
    level_of: np.ndarray
    perm: np.ndarray
    inv_perm: np.ndarray
    level_starts: np.ndarray
    width: int
    ell_cols: np.ndarray
    ell_vals: np.ndarray
    csr_rp: np.ndarray
    csr_ci: np.ndarray
    csr_v: np.ndarray


class Oracle:
    """The C restatement (hec_oracle.c)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_levels.restype = C.c_int
        L.orc_schedule.restype = C.c_int
        L.orc_hec_width.restype = C.c_int
        L.orc_hec_fill.restype = C.c_longlong
        L.orc_forward.restype = C.c_int
        L.orc_backward.restype = C.c_int
        L.orc_ilu0_inplace.restype = C.c_int
        L.orc_poisson7.restype = C.c_longlong
        L.orc_poisson27.restype = C.c_longlong
        L.orc_reservoir7.restype = C.c_longlong
        L.orc_reservoir7.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_ulonglong,
                                     P_int, P_int, P_dbl]
        L.orc_dot.restype = C.c_double

    # reference poisson.cpp:8-43
    def poisson7(self, nx, ny, nz) -> Csr:
        nnz = self.lib.orc_poisson7(nx, ny, nz, None, None, None)
        n = nx * ny * nz
        rp, ci, v = np.empty(n + 1, I32), np.empty(nnz, I32), np.empty(nnz, F64)
        self.lib.orc_poisson7(nx, ny, nz, _pi(rp), _pi(ci), _pd(v))
        return Csr(n, n, rp, ci, v)

    # SURVEY.md 8(d) C2 (27-point Poisson, the 7-point pattern of poisson.cpp:8-43 extended)
    def poisson27(self, nx, ny, nz) -> Csr:
        nnz = self.lib.orc_poisson27(nx, ny, nz, None, None, None)
        n = nx * ny * nz
        rp, ci, v = np.empty(n + 1, I32), np.empty(nnz, I32), np.empty(nnz, F64)
        self.lib.orc_poisson27(nx, ny, nz, _pi(rp), _pi(ci), _pd(v))
        return Csr(n, n, rp, ci, v)

    # SURVEY.md 8(d) C3 (heterogeneous reservoir 7-point)
    def reservoir7(self, nx, ny, nz, sigma=3.0, kz_ratio=0.1, seed=1606) -> Csr:
        nnz = self.lib.orc_reservoir7(nx, ny, nz, sigma, kz_ratio, seed, None, None, None)
        n = nx * ny * nz
        rp, ci, v = np.empty(n + 1, I32), np.empty(nnz, I32), np.empty(nnz, F64)
        self.lib.orc_reservoir7(nx, ny, nz, sigma, kz_ratio, seed, _pi(rp), _pi(ci), _pd(v))
        return Csr(n, n, rp, ci, v)

    # reference triangular.cpp:43-63
    def reverse(self, a: Csr) -> Csr:
        rp, ci, v = np.empty_like(a.rp), np.empty_like(a.ci), np.empty_like(a.v)
        self.lib.orc_reverse(a.n, _pi(a.rp), _pi(a.ci), _pd(a.v), _pi(rp), _pi(ci), _pd(v))
        return Csr(a.n, a.n, rp, ci, v)

    # reference triangular.cpp:65-88 (prepare_lower / prepare_upper)
    def prepare(self, t: Csr, upper=False, fixed_width: int = -1) -> Prepared:
        low = self.reverse(t) if upper else t
        n = low.n
        level = np.zeros(n, I32)
        nlev = self.lib.orc_levels(n, _pi(low.rp), _pi(low.ci), _pi(level))
        if nlev < 0:
            raise ValueError("oracle: not lower triangular")
        perm, inv, starts = np.empty(n, I32), np.empty(n, I32), np.empty(nlev + 1, I32)
        if self.lib.orc_schedule(n, _pi(level), nlev, _pi(perm), _pi(inv), _pi(starts)) < 0:
            raise ValueError("oracle: bad levels")
        rrp, rci, rv = np.empty_like(low.rp), np.empty_like(low.ci), np.empty_like(low.v)
        self.lib.orc_reorder(n, _pi(low.rp), _pi(low.ci), _pd(low.v), _pi(perm), _pi(inv), _pi(rrp), _pi(rci),
                             _pd(rv))
        w = self.lib.orc_hec_width(n, _pi(rrp), 1, fixed_width)
        cnnz = self.lib.orc_hec_fill(n, n, _pi(rrp), _pi(rci), _pd(rv), 1, w, None, None, None, None, None)
        if cnnz < 0:
            raise ValueError("oracle: missing diagonal")
        ec, ev = np.empty(w * n, I32), np.empty(w * n, F64)
        crp, cci, cv = np.empty(n + 1, I32), np.empty(cnnz, I32), np.empty(cnnz, F64)
        self.lib.orc_hec_fill(n, n, _pi(rrp), _pi(rci), _pd(rv), 1, w, _pi(ec), _pd(ev), _pi(crp), _pi(cci),
                              _pd(cv))
        return Prepared(int(upper), n, int(upper), nlev, level, perm, inv, starts, w, ec, ev, crp, cci, cv)

    # reference triangular.cpp:90-135 (Algorithm 2)
    def solve(self, p: Prepared, b) -> np.ndarray:
        b = np.ascontiguousarray(b, F64)
        x = np.empty(p.n, F64)
        self.lib.orc_solve(p.n, p.reversed, p.nlev, _pi(p.level_starts), _pi(p.perm), p.width, _pi(p.ell_cols),
                           _pd(p.ell_vals), _pi(p.csr_rp), _pi(p.csr_ci), _pd(p.csr_v), _pd(b), _pd(x))
        return x

    def forward(self, l: Csr, b) -> np.ndarray:
        b = np.ascontiguousarray(b, F64)
        x = np.empty(l.n, F64)
        if self.lib.orc_forward(l.n, _pi(l.rp), _pi(l.ci), _pd(l.v), _pd(b), _pd(x)) < 0:
            raise ValueError("oracle: not lower triangular with diagonal")
        return x

    def backward(self, u: Csr, b) -> np.ndarray:
        b = np.ascontiguousarray(b, F64)
        x = np.empty(u.n, F64)
        if self.lib.orc_backward(u.n, _pi(u.rp), _pi(u.ci), _pd(u.v), _pd(b), _pd(x)) < 0:
            raise ValueError("oracle: not upper triangular with diagonal")
        return x

    def spmv(self, a: Csr, x) -> np.ndarray:
        x = np.ascontiguousarray(x, F64)
        y = np.empty(a.n_rows, F64)
        self.lib.orc_spmv(a.n_rows, _pi(a.rp), _pi(a.ci), _pd(a.v), _pd(x), _pd(y))
        return y

    # reference ilu.cpp:23-79 (ilu0 = factor_on_pattern + split_factors)
    def ilu0(self, a: Csr):
        v = a.v.copy()
        dpos = np.empty(max(a.n, 1), I32)
        bad = C.c_int(-1)
        rc = self.lib.orc_ilu0_inplace(a.n, _pi(a.rp), _pi(a.ci), _pd(v), _pi(dpos), C.byref(bad))
        if rc < 0:
            raise ZeroDivisionError(f"oracle: zero pivot at row {bad.value}")
        n = a.n
        lrp, urp = [0], [0]
        lci, lv, uci, uv = [], [], [], []
        for i in range(n):
            s, d, e = a.rp[i], dpos[i], a.rp[i + 1]
            lci.extend(a.ci[s:d].tolist()); lv.extend(v[s:d].tolist())
            lci.append(i); lv.append(1.0)
            uci.extend(a.ci[d:e].tolist()); uv.extend(v[d:e].tolist())
            lrp.append(len(lci)); urp.append(len(uci))
        return (Csr(n, n, np.array(lrp, I32), np.array(lci, I32), np.array(lv, F64)),
                Csr(n, n, np.array(urp, I32), np.array(uci, I32), np.array(uv, F64)))

    # reference precond.cpp:119-145
    def apply(self, n, ext_rows, owned, pl: Prepared, pu: Prepared, r) -> np.ndarray:
        r = np.ascontiguousarray(r, F64)
        x = np.empty(n, F64)
        ext = np.ascontiguousarray(ext_rows, I32)
        own = np.ascontiguousarray(owned, np.int8)
        args = []
        for p in (pl, pu):
            args += [p.nlev, _pi(p.level_starts), _pi(p.perm), p.width, _pi(p.ell_cols), _pd(p.ell_vals),
                     _pi(p.csr_rp), _pi(p.csr_ci), _pd(p.csr_v)]
        self.lib.orc_apply(n, len(ext), _pi(ext), own.ctypes.data_as(P_chr), *args, _pd(r), _pd(x))
        return x

    def dot(self, a, b) -> float:
        a = np.ascontiguousarray(a, F64)
        b = np.ascontiguousarray(b, F64)
        return self.lib.orc_dot(len(a), _pd(a), _pd(b))


class RefError(RuntimeError):
    def __init__(self, code, msg, row=-1, block=-1):
        super().__init__(f"[{code}] {msg}")
        self.code, self.row, self.block = code, row, block


class Reference:
    """The reference library itself (oracle/_ref/libhecref.so via ref_shim.cpp)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: build it with `make -C oracle` where /root/reference exists")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        for name in ("ref_get_int", "ref_get_dbl", "ref_get_chr"):
            getattr(L, name).restype = C.c_longlong
        L.ref_rng_new.restype = C.c_void_p
        L.ref_rng_new.argtypes = [C.c_uint]
        L.ref_rng_free.argtypes = [C.c_void_p]
        L.ref_rng_int.restype = C.c_int
        L.ref_rng_int.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_rng_real.restype = C.c_double
        L.ref_rng_real.argtypes = [C.c_void_p, C.c_double, C.c_double]
        L.ref_random_vector.argtypes = [C.c_void_p, C.c_int, P_dbl]
        L.ref_random_matrix.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.POINTER(C.c_void_p)]
        L.ref_free.argtypes = [C.c_void_p]
        for name in ("ref_get_int", "ref_get_dbl", "ref_get_chr"):
            getattr(L, name).argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
        L.ref_prepare.argtypes = [C.c_int, P_int, P_int, P_dbl, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_solve.argtypes = [C.c_void_p, P_dbl, P_dbl, C.c_int]
        L.ref_apply.argtypes = [C.c_void_p, P_dbl, P_dbl, C.c_int]
        L.ref_precond.argtypes = [C.c_int, P_int, P_int, P_dbl, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                  C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_gmres.argtypes = [C.c_int, P_int, P_int, P_dbl, P_dbl, C.c_void_p, C.c_int, C.c_int, C.c_double,
                                C.c_double, C.c_int, P_dbl, P_dbl]
        L.ref_precond_single.argtypes = [C.c_int, P_int, P_int, P_dbl, P_int, P_int, P_dbl, C.POINTER(C.c_void_p)]
        L.ref_ilu.argtypes = [C.c_int, P_int, P_int, P_dbl, C.c_int, C.c_int, C.c_double, C.POINTER(C.c_void_p)]
        L.ref_prepared_from_arrays.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, P_int, P_int, P_int, P_int,
                                               C.c_int, P_int, P_dbl, P_int, P_int, P_dbl, C.POINTER(C.c_void_p)]

    def _check(self, rc):
        if rc != 0:
            L = self.lib
            raise RefError(rc, L.ref_last_error().decode(), L.ref_last_error_row(), L.ref_last_error_block())

    # --- bags
    class Bag:
        def __init__(self, ref, h):
            self.ref, self.h = ref, h

        def ints(self, name):
            p = C.POINTER(C.c_int)()
            n = self.ref.lib.ref_get_int(self.h, name.encode(), C.byref(p))
            if n < 0:
                raise KeyError(name)
            return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, I32)

        def dbls(self, name):
            p = C.POINTER(C.c_double)()
            n = self.ref.lib.ref_get_dbl(self.h, name.encode(), C.byref(p))
            if n < 0:
                raise KeyError(name)
            return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, F64)

        def chars(self, name):
            p = C.POINTER(C.c_char)()
            n = self.ref.lib.ref_get_chr(self.h, name.encode(), C.byref(p))
            if n < 0:
                raise KeyError(name)
            return np.frombuffer(C.string_at(p, n), dtype=np.int8).copy() if n else np.zeros(0, np.int8)

        def csr(self, prefix=""):
            d = self.ints(prefix + "dims")
            return Csr(int(d[0]), int(d[1]), self.ints(prefix + "rp"), self.ints(prefix + "ci"),
                       self.dbls(prefix + "v"))

        def prepared(self, prefix=""):
            m = self.ints(prefix + "meta")
            return Prepared(int(m[0]), int(m[1]), int(m[2]), int(m[3]), self.ints(prefix + "level_of"),
                            self.ints(prefix + "perm"), self.ints(prefix + "inv_perm"),
                            self.ints(prefix + "level_starts"), int(m[4]), self.ints(prefix + "ell_cols"),
                            self.dbls(prefix + "ell_vals"), self.ints(prefix + "csr_rp"),
                            self.ints(prefix + "csr_ci"), self.dbls(prefix + "csr_v"))

        def __del__(self):
            if self.h:
                self.ref.lib.ref_free(self.h)
                self.h = None

    def _bag(self, fn, *args):
        h = C.c_void_p()
        self._check(fn(*args, C.byref(h)))
        return Reference.Bag(self, h)

    # --- generators
    def poisson7(self, nx, ny, nz) -> Csr:
        return self._bag(self.lib.ref_poisson7, nx, ny, nz).csr()

    class Rng:
        """std::mt19937 plus the reference's test_helpers.hpp generators."""

        def __init__(self, ref, seed):
            self.ref, self.h = ref, ref.lib.ref_rng_new(seed)

        def uniform_int(self, lo, hi):
            return self.ref.lib.ref_rng_int(self.h, lo, hi)

        def uniform_real(self, lo, hi):
            return self.ref.lib.ref_rng_real(self.h, lo, hi)

        def vector(self, n):
            out = np.empty(n, F64)
            self.ref.lib.ref_random_vector(self.h, n, _pd(out))
            return out

        def matrix(self, kind, n, density):
            k = {"lower": 0, "upper": 1, "diag_dominant": 2}[kind]
            return self.ref._bag(self.ref.lib.ref_random_matrix, self.h, k, n, density).csr()

        def __del__(self):
            if self.h:
                self.ref.lib.ref_rng_free(self.h)
                self.h = None

    def rng(self, seed):
        return Reference.Rng(self, seed)

    # --- path
    def prepare(self, t: Csr, upper=False, fixed_width: Optional[int] = None):
        wm, w = (1, fixed_width) if fixed_width is not None else (0, 0)
        return self._bag(self.lib.ref_prepare, t.n, _pi(t.rp), _pi(t.ci), _pd(t.v), int(upper), wm, w)

    def prepared_from(self, p) -> "Reference.Bag":
        """A reference PreparedTriangular holding the given arrays (no setup)."""
        s, e = p.schedule, p.hec
        return self._bag(self.lib.ref_prepared_from_arrays, 1 if p.kind == "upper" else 0, p.n,
                         int(p.reversal_applied), s.nlev, _pi(np.ascontiguousarray(s.level_of, I32)),
                         _pi(np.ascontiguousarray(s.perm, I32)), _pi(np.ascontiguousarray(s.inv_perm, I32)),
                         _pi(np.ascontiguousarray(s.level_starts, I32)), e.ell.width,
                         _pi(np.ascontiguousarray(e.ell.col_indices, I32)),
                         _pd(np.ascontiguousarray(e.ell.values, F64)),
                         _pi(np.ascontiguousarray(e.csr_row_offsets, I32)),
                         _pi(np.ascontiguousarray(e.csr_col_indices, I32)),
                         _pd(np.ascontiguousarray(e.csr_values, F64)))

    def solve(self, prep_bag, b, workers=1) -> np.ndarray:
        b = np.ascontiguousarray(b, F64)
        x = np.empty_like(b)
        self._check(self.lib.ref_solve(prep_bag.h, _pd(b), _pd(x), workers))
        return x

    def serial_solve(self, t: Csr, b, upper=False) -> np.ndarray:
        b = np.ascontiguousarray(b, F64)
        x = np.empty_like(b)
        self._check(self.lib.ref_serial_solve(t.n, _pi(t.rp), _pi(t.ci), _pd(t.v), int(upper), _pd(b), _pd(x)))
        return x

    def spmv(self, a: Csr, x, workers=1) -> np.ndarray:
        x = np.ascontiguousarray(x, F64)
        y = np.empty(a.n_rows, F64)
        self._check(self.lib.ref_spmv(a.n_rows, a.n_cols, _pi(a.rp), _pi(a.ci), _pd(a.v), _pd(x), _pd(y), workers))
        return y

    def ilu(self, a: Csr, kind="ilu0", k_or_p=0, tol=0.0):
        bag = self._bag(self.lib.ref_ilu, a.n, _pi(a.rp), _pi(a.ci), _pd(a.v),
                        {"ilu0": 0, "iluk": 1, "ilut": 2}[kind], k_or_p, tol)
        return bag.csr("l_"), bag.csr("u_")

    def precond(self, a: Csr, kind, blocks, overlap, p=7, tol=0.1, fixed_width=None):
        wm, w = (1, fixed_width) if fixed_width is not None else (0, 0)
        return self._bag(self.lib.ref_precond, a.n, _pi(a.rp), _pi(a.ci), _pd(a.v),
                         {"bilu0": 0, "bilut": 1, "ras": 2}[kind], blocks, overlap, p, tol, wm, w)

    def precond_single(self, l: Csr, u: Csr):
        """One block holding the given factors (ILU(k) has no PrecondKind)."""
        return self._bag(self.lib.ref_precond_single, l.n, _pi(l.rp), _pi(l.ci), _pd(l.v), _pi(u.rp), _pi(u.ci),
                         _pd(u.v))

    def apply(self, bp_bag, r, workers=1) -> np.ndarray:
        r = np.ascontiguousarray(r, F64)
        x = np.empty_like(r)
        self._check(self.lib.ref_apply(bp_bag.h, _pd(r), _pd(x), workers))
        return x

    def gmres(self, a: Csr, b, bp_bag=None, restart=20, max_iters=10000, rel_tol=1e-6, abs_tol=0.0, workers=1):
        b = np.ascontiguousarray(b, F64)
        x = np.empty(a.n, F64)
        rep = np.zeros(5, F64)
        self._check(self.lib.ref_gmres(a.n, _pi(a.rp), _pi(a.ci), _pd(a.v), _pd(b), bp_bag.h if bp_bag else None,
                                       restart, max_iters, rel_tol, abs_tol, workers, _pd(x), _pd(rep)))
        return x, {"converged": bool(rep[0]), "iterations": int(rep[1]), "final_relative_residual": rep[2],
                   "solve_seconds": rep[3], "n_inner": int(rep[4])}


def load_oracle() -> Oracle:
    return Oracle()


def load_reference() -> Optional[Reference]:
    try:
        return Reference()
    except ImportError:
        return None
