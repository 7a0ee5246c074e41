"""Python mirror of the reference hecsolve API (proj/include/hecsolve/*.hpp).

Same names, argument meaning and error behaviour as the C++ drop-in; every
object is a thin owner of a C-ABI handle, arrays are zero-copy numpy views.
Host setup runs in the library's C++ (bit-identical to the reference); solve,
apply, and gmres run on the B200 through the C-ABI. Mapping of exceptions:
std::invalid_argument -> ValueError, std::out_of_range -> IndexError,
hec::ZeroPivotError -> ZeroPivotError(row, block), CUDA/runtime -> HecError.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import ZeroPivotError, HecError, check, lib  # noqa: F401

_i32 = np.int32
_f64 = np.float64


def _p_int(a):
    return a.ctypes.data_as(L.P_int) if a is not None else None


def _p_dbl(a):
    return a.ctypes.data_as(L.P_dbl) if a is not None else None


def _view(ptr, count, dtype):
    if count == 0 or not ptr:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(count,)).view(dtype)


def _f64_vec(x, n=None, name="vector"):
    a = np.ascontiguousarray(x, dtype=_f64)
    if a.ndim != 1 or (n is not None and a.shape[0] != n):
        raise ValueError(f"{name}: dimension mismatch")
    return a


# ----------------------------------------------------------------- CSR ----
class CsrMatrix:
    """hec::CsrMatrix (reference csr.hpp:17-27). Owns a C++ matrix."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        nr, nc, nnz = C.c_int(), C.c_int(), C.c_longlong()
        rp, ci, v = L.P_int(), L.P_int(), L.P_dbl()
        check(lib.hec_csr_view(self._h, C.byref(nr), C.byref(nc), C.byref(nnz), C.byref(rp), C.byref(ci),
                               C.byref(v)))
        self.n_rows, self.n_cols = nr.value, nc.value
        self.row_offsets = _view(rp, self.n_rows + 1, _i32)
        self.col_indices = _view(ci, nnz.value, _i32)
        self.values = _view(v, nnz.value, _f64)

    @classmethod
    def from_arrays(cls, n_rows, n_cols, row_offsets, col_indices, values):
        rp = np.ascontiguousarray(row_offsets, dtype=_i32)
        ci = np.ascontiguousarray(col_indices, dtype=_i32)
        v = np.ascontiguousarray(values, dtype=_f64)
        if rp.shape[0] != n_rows + 1:
            raise ValueError("CsrMatrix: row_offsets must have n_rows + 1 entries")
        h = C.c_void_p()
        check(lib.hec_csr_create(n_rows, n_cols, _p_int(rp), _p_int(ci), _p_dbl(v), C.byref(h)))
        return cls(h)

    @property
    def handle(self):
        return self._h

    def nnz(self) -> int:
        return int(self.col_indices.shape[0])

    def __eq__(self, other):
        return (isinstance(other, CsrMatrix) and self.n_rows == other.n_rows and self.n_cols == other.n_cols
                and np.array_equal(self.row_offsets, other.row_offsets)
                and np.array_equal(self.col_indices, other.col_indices)
                and np.array_equal(self.values.view(np.uint64), other.values.view(np.uint64)))

    def __del__(self):
        if getattr(self, "_h", None):
            lib.hec_csr_destroy(self._h)
            self._h = None


def csr_from_triples(n_rows: int, n_cols: int, triples) -> CsrMatrix:
    """Reference csr.cpp:9-41: sorted, duplicates and out-of-range rejected."""
    t = list(triples)
    rows = np.array([a for a, _, _ in t], dtype=_i32)
    cols = np.array([b for _, b, _ in t], dtype=_i32)
    vals = np.array([c for _, _, c in t], dtype=_f64)
    h = C.c_void_p()
    check(lib.hec_csr_from_triples(n_rows, n_cols, len(t), _p_int(rows), _p_int(cols), _p_dbl(vals), C.byref(h)))
    return CsrMatrix(h)


def spmv_csr(a: CsrMatrix, x, workers: int = 1) -> np.ndarray:
    """Host y = A x (utility for right-hand sides; reference csr.cpp:43-57)."""
    xv = _f64_vec(x, a.n_cols, "spmv_csr")
    y = np.empty(a.n_rows, dtype=_f64)
    check(lib.hec_csr_spmv_host(a.handle, _p_dbl(xv), _p_dbl(y), workers))
    return y


def _gen(fn, *args) -> CsrMatrix:
    h = C.c_void_p()
    check(fn(*args, C.byref(h)))
    return CsrMatrix(h)


def gen_poisson7(nx, ny, nz) -> CsrMatrix:
    return _gen(lib.hec_gen_poisson7, nx, ny, nz)


def gen_poisson27(nx, ny, nz) -> CsrMatrix:
    return _gen(lib.hec_gen_poisson27, nx, ny, nz)


def gen_reservoir7(nx, ny, nz, sigma=3.0, kz_ratio=0.1, seed=1606) -> CsrMatrix:
    return _gen(lib.hec_gen_reservoir7, nx, ny, nz, sigma, kz_ratio, seed)


def permute_symmetric(a: CsrMatrix, perm) -> CsrMatrix:
    p = np.ascontiguousarray(perm, dtype=_i32)
    return _gen(lib.hec_permute_symmetric, a.handle, _p_int(p))


def csr_submatrix(a: CsrMatrix, rows) -> CsrMatrix:
    """Principal submatrix on ascending `rows` (reference precond.cpp:13-34)."""
    r = np.ascontiguousarray(rows, dtype=_i32)
    h = C.c_void_p()
    check(lib.hec_csr_submatrix(a.handle, _p_int(r), r.shape[0], C.byref(h)))
    return CsrMatrix(h)


def partition(a: CsrMatrix, parts: int, overlap: int):
    """hec::partition_graph + hec::extend_overlap (reference partition.cpp:28-107).
    Returns (part_of[n], [ascending extended rows of part p for p < parts])."""
    h = C.c_void_p()
    check(lib.hec_partition_create(a.handle, parts, overlap, C.byref(h)))
    try:
        n, np_ = C.c_int(), C.c_int()
        po, eo, er = L.P_int(), L.P_int(), L.P_int()
        check(lib.hec_partition_view(h, C.byref(n), C.byref(np_), C.byref(po), C.byref(eo), C.byref(er)))
        part_of = _view(po, n.value, _i32).copy()
        offs = _view(eo, np_.value + 1, _i32).copy()
        rows = _view(er, int(offs[-1]), _i32).copy()
        return part_of, [rows[offs[p]:offs[p + 1]] for p in range(np_.value)]
    finally:
        lib.hec_partition_destroy(h)


class Krylov:
    """The fused Krylov vector kernels (hec_krylov_*), device pointers / tensors."""

    def __init__(self, n: int):
        self.n = n
        self._h = C.c_void_p()
        check(lib.hec_krylov_create(n, C.byref(self._h)))

    def mgs(self, w, v_prev, h_prev, v_next, out, stream=None):
        check(lib.hec_krylov_mgs(self._h, C.c_void_p(_ptr(w)), C.c_void_p(_ptr(v_prev) if v_prev is not None else None),
                                 C.c_void_p(_ptr(h_prev) if h_prev is not None else None),
                                 C.c_void_p(_ptr(v_next)), C.c_void_p(_ptr(out)), C.c_void_p(_stream(stream))))

    def scale(self, y, x, s, stream=None):
        check(lib.hec_krylov_scale(self._h, C.c_void_p(_ptr(y)), C.c_void_p(_ptr(x)), C.c_void_p(_ptr(s)),
                                   C.c_void_p(_stream(stream))))

    def combine(self, j, xc, V, ldv, y, stream=None):
        check(lib.hec_krylov_combine(self._h, j, C.c_void_p(_ptr(xc)), C.c_void_p(_ptr(V)), ldv,
                                     C.c_void_p(_ptr(y)), C.c_void_p(_stream(stream))))

    def add(self, x, d, stream=None):
        check(lib.hec_krylov_add(self._h, C.c_void_p(_ptr(x)), C.c_void_p(_ptr(d)), C.c_void_p(_stream(stream))))

    def sqrt(self, a, out, stream=None):
        check(lib.hec_krylov_sqrt(self._h, C.c_void_p(_ptr(a)), C.c_void_p(_ptr(out)), C.c_void_p(_stream(stream))))

    def __del__(self):
        if getattr(self, "_h", None):
            lib.hec_krylov_destroy(self._h)
            self._h = None


def random_ordering(n, seed=1606) -> np.ndarray:
    p = np.empty(n, dtype=_i32)
    check(lib.hec_random_ordering(n, seed, _p_int(p)))
    return p


def rcm_ordering(a: CsrMatrix) -> np.ndarray:
    p = np.empty(a.n_rows, dtype=_i32)
    check(lib.hec_rcm_ordering(a.handle, _p_int(p)))
    return p


# ----------------------------------------------------------------- ILU ----
@dataclass
class IluFactors:
    l: CsrMatrix
    u: CsrMatrix
    n: int


def _ilu(fn, a, *args) -> IluFactors:
    hl, hu = C.c_void_p(), C.c_void_p()
    check(fn(a.handle, *args, C.byref(hl), C.byref(hu)))
    return IluFactors(CsrMatrix(hl), CsrMatrix(hu), a.n_rows)


def ilu0(a: CsrMatrix) -> IluFactors:
    return _ilu(lib.hec_ilu0, a)


def ilu_k(a: CsrMatrix, k: int) -> IluFactors:
    return _ilu(lib.hec_ilu_k, a, k)


def ilut(a: CsrMatrix, p: int, tol: float) -> IluFactors:
    return _ilu(lib.hec_ilut, a, p, tol)


# ---------------------------------------------------------- triangular ----
@dataclass(frozen=True)
class WidthPolicy:
    """Reference hec.hpp:25-33."""
    mode: str = "automatic"
    width: int = 0

    @staticmethod
    def fixed(w: int) -> "WidthPolicy":
        return WidthPolicy("fixed", w)

    @staticmethod
    def automatic() -> "WidthPolicy":
        return WidthPolicy()

    def c_args(self):
        return (1, self.width) if self.mode == "fixed" else (0, 0)


@dataclass
class LevelSchedule:
    n: int
    nlev: int
    level_of: np.ndarray
    perm: np.ndarray
    inv_perm: np.ndarray
    level_starts: np.ndarray


@dataclass
class EllMatrix:
    n_rows: int
    width: int
    col_indices: np.ndarray
    values: np.ndarray


@dataclass
class HecMatrix:
    n_rows: int
    n_cols: int
    ell: EllMatrix
    csr_row_offsets: np.ndarray
    csr_col_indices: np.ndarray
    csr_values: np.ndarray
    _handle: object = None  # owning hec_hec_t when built by hec_from_csr

    def __del__(self):
        if self._handle is not None:
            lib.hec_hec_destroy(self._handle)
            self._handle = None


def hec_from_csr(a: CsrMatrix, triangular: bool = False, policy: "Optional[WidthPolicy]" = None) -> HecMatrix:
    """hec::hec_from_csr (reference hec.hpp:48, hec.cpp:28-86), host setup."""
    mode, width = (policy or WidthPolicy()).c_args()
    h = C.c_void_p()
    check(lib.hec_hec_from_csr(a.handle, int(bool(triangular)), mode, width, C.byref(h)))
    v = L.HecView()
    check(lib.hec_hec_view_get(h, C.byref(v)))
    n, w = v.n_rows, v.ell_width
    return HecMatrix(n, v.n_cols, EllMatrix(n, w, _view(v.ell_cols, w * n, _i32), _view(v.ell_vals, w * n, _f64)),
                     _view(v.csr_row_offsets, n + 1, _i32), _view(v.csr_cols, v.csr_nnz, _i32),
                     _view(v.csr_vals, v.csr_nnz, _f64), h)


def spmv_hec(h: HecMatrix, x, workers: int = 1) -> np.ndarray:
    """hec::spmv_hec on the B200 (reference hec.cpp:88-108); h from hec_from_csr."""
    if h._handle is None:
        raise ValueError("spmv_hec: HecMatrix not built by hec_from_csr")
    xv = _f64_vec(x, h.n_cols, "spmv_hec")
    y = np.empty(h.n_rows, dtype=_f64)
    check(lib.hec_hec_spmv_host(h._handle, _p_dbl(xv), _p_dbl(y), workers))
    return y


class PreparedTriangular:
    """hec::PreparedTriangular (reference triangular.hpp:18-24); views are zero-copy."""

    def __init__(self, handle, owner=None):
        self._h = handle
        self._owner = owner  # keeps a borrowed handle's parent alive
        v = L.PrepView()
        check(lib.hec_prep_view_get(self._h, C.byref(v)))
        n, nlev, w = v.n, v.nlev, v.ell_width
        self.kind = "upper" if v.kind else "lower"
        self.n = n
        self.reversal_applied = bool(v.reversal_applied)
        self.schedule = LevelSchedule(n, nlev, _view(v.level_of, n, _i32), _view(v.perm, n, _i32),
                                      _view(v.inv_perm, n, _i32), _view(v.level_starts, nlev + 1, _i32))
        self.hec = HecMatrix(n, n, EllMatrix(n, w, _view(v.ell_cols, w * n, _i32), _view(v.ell_vals, w * n, _f64)),
                             _view(v.csr_row_offsets, n + 1, _i32), _view(v.csr_cols, v.csr_nnz, _i32),
                             _view(v.csr_vals, v.csr_nnz, _f64))

    @property
    def handle(self):
        return self._h

    def device(self) -> "DeviceTri":
        """The device triangle cached inside this object (built on first use)."""
        t = C.c_void_p()
        check(lib.hec_prep_device(self._h, C.byref(t)))
        return DeviceTri(t, owner=self)

    def __del__(self):
        if getattr(self, "_h", None) and self._owner is None:
            lib.hec_prep_destroy(self._h)
        self._h = None


def _prepare(t: CsrMatrix, upper: int, policy: Optional[WidthPolicy]) -> PreparedTriangular:
    mode, width = (policy or WidthPolicy()).c_args()
    h = C.c_void_p()
    check(lib.hec_prepare(t.handle, upper, mode, width, C.byref(h)))
    return PreparedTriangular(h)


def prepare_lower(l: CsrMatrix, policy: Optional[WidthPolicy] = None) -> PreparedTriangular:
    return _prepare(l, 0, policy)


def prepare_upper(u: CsrMatrix, policy: Optional[WidthPolicy] = None) -> PreparedTriangular:
    return _prepare(u, 1, policy)


def solve(p: PreparedTriangular, b, workers: int = 1) -> np.ndarray:
    """hec::solve on the B200 (reference triangular.cpp:90-135); workers ignored."""
    bv = _f64_vec(b, None, "solve")
    if bv.shape[0] != p.n:
        raise ValueError("solve: dimension mismatch")
    x = np.empty(p.n, dtype=_f64)
    check(lib.hec_prep_solve_host(p.handle, _p_dbl(bv), _p_dbl(x)))
    return x


def serial_forward_solve(l: CsrMatrix, b) -> np.ndarray:
    bv = _f64_vec(b, l.n_rows, "serial_forward_solve")
    x = np.empty(l.n_rows, dtype=_f64)
    check(lib.hec_serial_solve(l.handle, 0, _p_dbl(bv), _p_dbl(x)))
    return x


def serial_backward_solve(u: CsrMatrix, b) -> np.ndarray:
    bv = _f64_vec(b, u.n_rows, "serial_backward_solve")
    x = np.empty(u.n_rows, dtype=_f64)
    check(lib.hec_serial_solve(u.handle, 1, _p_dbl(bv), _p_dbl(x)))
    return x


# ------------------------------------------------------- device objects ----
def _ptr(t) -> int:
    """Raw device pointer of a torch tensor / int / None."""
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    return int(t.data_ptr())


def _stream(s) -> Optional[int]:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return int(s.cuda_stream)


class DeviceTri:
    """hec_tri_t: a device-resident prepared triangle."""

    def __init__(self, handle, owner=None):
        self._h = handle
        self._owner = owner

    @classmethod
    def create(cls, p: PreparedTriangular, strategy=L.STRATEGY_AUTO, ctas=0, threads=0) -> "DeviceTri":
        s = p.schedule
        e = p.hec
        opt = L.TriOptions(strategy, ctas, threads)
        h = C.c_void_p()
        check(lib.hec_tri_create(p.n, int(p.reversal_applied), s.nlev, _p_int(s.level_starts), _p_int(s.inv_perm),
                                 e.ell.width, _p_int(e.ell.col_indices), _p_dbl(e.ell.values),
                                 _p_int(e.csr_row_offsets), _p_int(e.csr_col_indices), _p_dbl(e.csr_values),
                                 C.byref(opt), C.byref(h)))
        return cls(h)

    def solve(self, b_dev, x_dev, stream=None) -> None:
        check(lib.hec_tri_solve(self._h, C.c_void_p(_ptr(b_dev)), C.c_void_p(_ptr(x_dev)),
                                C.c_void_p(_stream(stream)) if stream is not None else None))

    def permute_in(self, b_dev, bp_dev, stream=None) -> None:
        """bp in the layout's private order; bp holds info()["wave_len"] + 2 doubles."""
        check(lib.hec_tri_permute_in(self._h, C.c_void_p(_ptr(b_dev)), C.c_void_p(_ptr(bp_dev)),
                                     C.c_void_p(_stream(stream)) if stream is not None else None))

    def solve_ordered(self, bp_dev, x_dev, stream=None) -> None:
        """The solve from a right-hand side already in reordered-row order."""
        check(lib.hec_tri_solve_ordered(self._h, C.c_void_p(_ptr(bp_dev)), C.c_void_p(_ptr(x_dev)),
                                        C.c_void_p(_stream(stream)) if stream is not None else None))

    def solve_wave(self, bp_dev, xw_dev, stream=None) -> None:
        """The solve alone, x left in the layout's wave order (see permute_out)."""
        check(lib.hec_tri_solve_wave(self._h, C.c_void_p(_ptr(bp_dev)), C.c_void_p(_ptr(xw_dev)),
                                     C.c_void_p(_stream(stream)) if stream is not None else None))

    def permute_out(self, xw_dev, x_dev, stream=None) -> None:
        """x[o] = xw[wpos[o]]: the solution order from solve_wave's output."""
        check(lib.hec_tri_permute_out(self._h, C.c_void_p(_ptr(xw_dev)), C.c_void_p(_ptr(x_dev)),
                                      C.c_void_p(_stream(stream)) if stream is not None else None))

    def solve_host(self, b) -> np.ndarray:
        bv = _f64_vec(b, None, "solve")
        x = np.empty_like(bv)
        check(lib.hec_tri_solve_host(self._h, _p_dbl(bv), _p_dbl(x)))
        return x

    def info(self) -> dict:
        i = L.TriInfo()
        check(lib.hec_tri_query(self._h, C.byref(i)))
        return i.as_dict()

    def solve_traced(self, b_dev, x_dev, stream=None):
        """Diagnostics: run one solve and return (trace[chunks, 8] uint64, cta_chunk0)."""
        import torch
        info = self.info()
        trace = torch.zeros(max(info["chunks"], 1) * 64, dtype=torch.int64, device="cuda")
        c0 = np.zeros(info["ctas"] + 1, dtype=_i32)
        check(lib.hec_tri_solve_traced(self._h, C.c_void_p(_ptr(b_dev)), C.c_void_p(_ptr(x_dev)),
                                       C.c_void_p(_stream(stream)) if stream is not None else None,
                                       C.c_void_p(_ptr(trace)), _p_int(c0)))
        torch.cuda.synchronize()
        return trace.cpu().numpy().view(np.uint64).reshape(-1, 64)[:info["chunks"]], c0

    def __del__(self):
        if getattr(self, "_h", None) and self._owner is None:
            lib.hec_tri_destroy(self._h)
        self._h = None


class DevicePrecond:
    """hec_precond_t: L+U pair with RAS gather/scatter."""

    def __init__(self, handle, owner=None):
        self._h = handle
        self._owner = owner

    @classmethod
    def create(cls, n, pl: PreparedTriangular, pu: PreparedTriangular, gather=None, owned=None,
               strategy=L.STRATEGY_AUTO, ctas=0, threads=0):
        opt = L.TriOptions(strategy, ctas, threads)
        g = None if gather is None else np.ascontiguousarray(gather, dtype=_i32)
        o = None if owned is None else np.ascontiguousarray(owned, dtype=np.int8)
        h = C.c_void_p()
        args = []
        for p in (pl, pu):
            s, e = p.schedule, p.hec
            args += [s.nlev, _p_int(s.level_starts), _p_int(s.inv_perm), e.ell.width, _p_int(e.ell.col_indices),
                     _p_dbl(e.ell.values), _p_int(e.csr_row_offsets), _p_int(e.csr_col_indices),
                     _p_dbl(e.csr_values)]
        check(lib.hec_precond_create(n, pl.n, _p_int(g), o.ctypes.data_as(L.P_char) if o is not None else None,
                                     *args, C.byref(opt), C.byref(h)))
        return cls(h)

    @classmethod
    def create_local(cls, n_in, n_out, pl: PreparedTriangular, pu: PreparedTriangular, gather, out_index,
                     strategy=L.STRATEGY_AUTO, ctas=0, threads=0):
        """One RAS subdomain of a distributed vector: factor row k reads r[gather[k]]
        and writes x[out_index[k]] (skipped when negative); see hec_precond_create_local."""
        opt = L.TriOptions(strategy, ctas, threads)
        g = np.ascontiguousarray(gather, dtype=_i32)
        o = np.ascontiguousarray(out_index, dtype=_i32)
        if g.shape[0] != pl.n or o.shape[0] != pl.n:
            raise ValueError("create_local: map size must equal the factor size")
        h = C.c_void_p()
        args = []
        for p in (pl, pu):
            s, e = p.schedule, p.hec
            args += [s.nlev, _p_int(s.level_starts), _p_int(s.inv_perm), e.ell.width, _p_int(e.ell.col_indices),
                     _p_dbl(e.ell.values), _p_int(e.csr_row_offsets), _p_int(e.csr_col_indices),
                     _p_dbl(e.csr_values)]
        check(lib.hec_precond_create_local(n_in, n_out, pl.n, _p_int(g), _p_int(o), *args, C.byref(opt),
                                           C.byref(h)))
        return cls(h)

    def apply(self, r_dev, x_dev, stream=None) -> None:
        check(lib.hec_precond_apply(self._h, C.c_void_p(_ptr(r_dev)), C.c_void_p(_ptr(x_dev)),
                                    C.c_void_p(_stream(stream)) if stream is not None else None))

    def apply_host(self, r) -> np.ndarray:
        rv = _f64_vec(r, None, "apply")
        x = np.empty_like(rv)
        check(lib.hec_precond_apply_host(self._h, _p_dbl(rv), _p_dbl(x)))
        return x

    def info(self):
        a, b = L.TriInfo(), L.TriInfo()
        check(lib.hec_precond_query(self._h, C.byref(a), C.byref(b)))
        return a.as_dict(), b.as_dict()

    def __del__(self):
        if getattr(self, "_h", None) and self._owner is None:
            lib.hec_precond_destroy(self._h)
        self._h = None


class DeviceSpmv:
    """hec_spmv_t: the device HEC SpMV (from CSR: bitwise spmv_csr; from_hec: bitwise spmv_hec)."""

    def __init__(self, a: Optional[CsrMatrix], _h=None, _dims=None):
        if a is None:
            self._h = _h
            self.n_rows, self.n_cols = _dims
            return
        self.n_rows, self.n_cols = a.n_rows, a.n_cols
        h = C.c_void_p()
        check(lib.hec_spmv_create(a.n_rows, a.n_cols, _p_int(a.row_offsets), _p_int(a.col_indices),
                                  _p_dbl(a.values), C.byref(h)))
        self._h = h

    @classmethod
    def from_hec(cls, m: HecMatrix) -> "DeviceSpmv":
        h = C.c_void_p()
        e = m.ell
        check(lib.hec_spmv_create_hec(m.n_rows, m.n_cols, e.width, _p_int(e.col_indices), _p_dbl(e.values),
                                      _p_int(m.csr_row_offsets), _p_int(m.csr_col_indices),
                                      _p_dbl(m.csr_values), C.byref(h)))
        return cls(None, h, (m.n_rows, m.n_cols))

    def residual(self, b_dev, x_dev, y_dev, stream=None):
        """y = b - A x"""
        check(lib.hec_spmv_residual(self._h, C.c_void_p(_ptr(b_dev)), C.c_void_p(_ptr(x_dev)),
                                    C.c_void_p(_ptr(y_dev)),
                                    C.c_void_p(_stream(stream)) if stream is not None else None))

    def run(self, x_dev, y_dev, stream=None):
        check(lib.hec_spmv_run(self._h, C.c_void_p(_ptr(x_dev)), C.c_void_p(_ptr(y_dev)),
                               C.c_void_p(_stream(stream)) if stream is not None else None))

    def run_host(self, x) -> np.ndarray:
        xv = _f64_vec(x, self.n_cols, "spmv")
        y = np.empty(self.n_rows, dtype=_f64)
        check(lib.hec_spmv_run_host(self._h, _p_dbl(xv), _p_dbl(y)))
        return y

    def __del__(self):
        if getattr(self, "_h", None):
            lib.hec_spmv_destroy(self._h)
        self._h = None


# ----------------------------------------------------- preconditioners ----
PRECOND_KINDS = {"bilu0": 0, "bilut": 1, "ras": 2, "biluk": 3}


class BlockPreconditioner:
    """hec::BlockPreconditioner (reference precond.hpp:20-31)."""

    def __init__(self, handle, kind):
        self._h = handle
        self.kind = kind
        n, parts, n_ext = C.c_int(), C.c_int(), C.c_int()
        check(lib.hec_bp_dims(self._h, C.byref(n), C.byref(parts), C.byref(n_ext)))
        self.n, self.n_parts, self.n_ext = n.value, parts.value, n_ext.value
        self.part_of = np.empty(self.n, dtype=_i32)
        self.offsets = np.empty(self.n_parts + 1, dtype=_i32)
        self.ext_rows = np.empty(self.n_ext, dtype=_i32)
        self.owned = np.empty(self.n_ext, dtype=np.int8)
        check(lib.hec_bp_maps(self._h, _p_int(self.part_of), _p_int(self.offsets), _p_int(self.ext_rows),
                              self.owned.ctypes.data_as(L.P_char)))
        hl, hu = C.c_void_p(), C.c_void_p()
        check(lib.hec_bp_prepared(self._h, C.byref(hl), C.byref(hu)))
        self.prepared_l = PreparedTriangular(hl, owner=self)
        self.prepared_u = PreparedTriangular(hu, owner=self)

    @property
    def handle(self):
        return self._h

    @property
    def extended_parts(self):
        return [self.ext_rows[self.offsets[p]:self.offsets[p + 1]] for p in range(self.n_parts)]

    @property
    def parts(self):
        return [np.flatnonzero(self.part_of == p).astype(_i32) for p in range(self.n_parts)]

    @property
    def restriction(self):
        return [self.owned[self.offsets[p]:self.offsets[p + 1]] for p in range(self.n_parts)]

    def device(self) -> DevicePrecond:
        d = C.c_void_p()
        check(lib.hec_bp_device(self._h, C.byref(d)))
        return DevicePrecond(d, owner=self)

    def __del__(self):
        if getattr(self, "_h", None):
            self.prepared_l = self.prepared_u = None
            lib.hec_bp_destroy(self._h)
        self._h = None


def build_preconditioner(a: CsrMatrix, kind: str, blocks: int, overlap: int, ilut_p: int = 7,
                         ilut_tol: float = 0.1, policy: Optional[WidthPolicy] = None,
                         fill_level: int = 1) -> BlockPreconditioner:
    mode, width = (policy or WidthPolicy()).c_args()
    h = C.c_void_p()
    check(lib.hec_bp_build(a.handle, PRECOND_KINDS[kind], blocks, overlap, ilut_p, ilut_tol, mode, width,
                           fill_level, C.byref(h)))
    return BlockPreconditioner(h, kind)


def apply(m: BlockPreconditioner, r, workers: int = 1) -> np.ndarray:
    """hec::apply on the B200 (reference precond.cpp:119-145)."""
    rv = _f64_vec(r, None, "apply")
    if rv.shape[0] != m.n:
        raise ValueError("apply: dimension mismatch")
    x = np.empty(m.n, dtype=_f64)
    check(lib.hec_bp_apply_host(m.handle, _p_dbl(rv), _p_dbl(x)))
    return x


# --------------------------------------------------------------- GMRES ----
@dataclass
class SolverConfig:
    restart: int = 20
    max_iters: int = 10000
    rel_tol: float = 1e-6
    abs_tol: float = 0.0


@dataclass
class SolveReport:
    converged: bool = False
    iterations: int = 0
    final_relative_residual: float = 0.0
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0
    inner_residuals: list = field(default_factory=list)


@dataclass
class SolveResult:
    x: np.ndarray
    report: SolveReport


def gmres(a: CsrMatrix, b, m: Optional[BlockPreconditioner], cfg: SolverConfig = SolverConfig(),
          workers: int = 1) -> SolveResult:
    """hec::gmres with device SpMV / apply / Krylov ops (reference gmres.cpp:28-137)."""
    bv = _f64_vec(b, None, "gmres")
    x = np.empty(a.n_rows, dtype=_f64)
    rep = L.GmresReport()
    cap = max(cfg.max_iters, 0) + 1
    inner = np.empty(cap, dtype=_f64)
    c = L.GmresConfig(cfg.restart, cfg.max_iters, cfg.rel_tol, cfg.abs_tol)
    check(lib.hec_gmres_host(a.handle, _p_dbl(bv), m.handle if m is not None else None, C.byref(c), _p_dbl(x),
                             C.byref(rep), _p_dbl(inner), cap))
    r = SolveReport(bool(rep.converged), rep.iterations, rep.final_relative_residual, 0.0, rep.solve_seconds,
                    inner[:min(rep.n_inner, cap)].tolist())
    return SolveResult(x, r)


def device_available() -> bool:
    return bool(lib.hec_device_available())
