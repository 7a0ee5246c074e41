"""Device HEC SpMV (spmv_hec.cu) against the reference's loops, bit for bit.

* from CSR (hec_spmv_create; the layout GMRES multiplies with): spmv_csr,
  proj/src/csr.cpp:43-57 -- the C oracle's orc_spmv and the reference library;
* from a HecMatrix (hec_spmv_create_hec, and the drop-in hec::spmv_hec):
  proj/src/hec.cpp:88-108 -- ELL slots 0..w-1 including the padding products,
  then the CSR part in storage order, restated below with numpy elementwise
  IEEE operations (no FMA);
* the fused residual y = b - A x (gmres.cpp:19-24).
Widths cover pure-CSR (w = 0), mostly-remainder (w = 1), the automatic median
and heavy padding (w = 32); sizes cover empty, one row, n not a multiple of the
64-row warp tile, rows far longer than a 128-entry staging tile, and 256^3.
"""
import numpy as np
import pytest

from golden_util import load
from util import bits_equal, random_diag_dominant, to_oracle, to_product

pytestmark = pytest.mark.gpu


def hec_reference(h, x):
    """spmv_hec restated (hec.cpp:88-108): acc = 0; acc += v*x[c] per ELL slot, then per CSR entry."""
    n, w = h.n_rows, h.ell.width
    x = np.asarray(x, np.float64)
    acc = np.zeros(n)
    cols = np.asarray(h.ell.col_indices).reshape(w, n) if w else np.zeros((0, n), np.int32)
    vals = np.asarray(h.ell.values).reshape(w, n) if w else np.zeros((0, n))
    for k in range(w):
        acc = acc + vals[k] * x[cols[k]]
    rp = np.asarray(h.csr_row_offsets, np.int64)
    ci, cv = np.asarray(h.csr_col_indices), np.asarray(h.csr_values)
    lens = rp[1:] - rp[:-1]
    for j in range(int(lens.max()) if n else 0):
        m = lens > j
        e = rp[:-1][m] + j
        acc[m] = acc[m] + cv[e] * x[ci[e]]
    return acc


def long_rows(rng, n=700):
    """Rows of very different lengths (some > 300 entries): the staged remainder path."""
    from oracle.oracle import Csr
    rp, ci, v = [0], [], []
    for i in range(n):
        k = int(rng.integers(0, 400)) if i % 37 == 0 else int(rng.integers(0, 9))
        cols = np.sort(rng.choice(n, size=min(k, n), replace=False))
        ci.extend(cols.tolist())
        v.extend(rng.uniform(-1, 1, len(cols)).tolist())
        rp.append(len(ci))
    return Csr(n, n, np.array(rp), np.array(ci), np.array(v))


def matrices(H):
    rng = np.random.default_rng(2024)
    return [H.gen_poisson7(17, 13, 11), H.gen_poisson27(9, 8, 7), H.gen_reservoir7(10, 9, 8),
            to_product(H, random_diag_dominant(300, 0.05, rng)), to_product(H, long_rows(rng)),
            H.csr_from_triples(1, 1, [(0, 0, 2.0)]), H.csr_from_triples(65, 65, [(i, i, 1.0 + i) for i in range(65)]),
            H.csr_from_triples(3, 5, [(0, 4, 1.0), (2, 0, -2.0)])]


def test_from_csr_bitwise_vs_spmv_csr(H, orc, ref):
    for a in matrices(H):
        x = np.random.default_rng(1).uniform(-1, 1, a.n_cols)
        want = orc.spmv(to_oracle(a), x)
        assert bits_equal(want, ref.spmv(to_oracle(a), x))
        assert bits_equal(H.DeviceSpmv(a).run_host(x), want)
        assert bits_equal(H.spmv_csr(a, x), want)  # the drop-in hec::spmv_csr


def test_from_hec_bitwise_vs_spmv_hec(H):
    for a in matrices(H):
        x = np.random.default_rng(2).uniform(-1, 1, a.n_cols)
        for policy in (None, H.WidthPolicy.fixed(0), H.WidthPolicy.fixed(1), H.WidthPolicy.fixed(32)):
            h = H.hec_from_csr(a, False, policy)
            want = hec_reference(h, x)
            assert bits_equal(H.DeviceSpmv.from_hec(h).run_host(x), want)
            assert bits_equal(H.spmv_hec(h, x), want)
            if a.n_rows == a.n_cols:
                assert bits_equal(want, H.spmv_csr(a, x))  # HEC of the same CSR: same sums


def test_hec_padding_multiplied_like_the_reference(H):
    # padding slots multiply x[min(i, n_cols-1)] (hec.cpp:69,99-102): an Inf there turns a
    # padded row into NaN in the reference, and so on the device
    a = H.csr_from_triples(4, 4, [(0, 0, 1.0), (0, 1, 2.0), (1, 1, 3.0), (2, 2, 4.0), (2, 3, 1.0), (3, 3, 5.0)])
    h = H.hec_from_csr(a, False, H.WidthPolicy.fixed(2))
    x = np.array([1.0, np.inf, 2.0, 3.0])
    want = hec_reference(h, x)
    got = H.spmv_hec(h, x)
    assert bits_equal(got, want) and np.isnan(got[1])
    # the CSR-built layout skips padding: spmv_csr semantics
    assert bits_equal(H.DeviceSpmv(a).run_host(x), orc_like_csr(a, x))


def orc_like_csr(a, x):
    rp, ci, v = np.asarray(a.row_offsets), np.asarray(a.col_indices), np.asarray(a.values)
    y = np.zeros(a.n_rows)
    for i in range(a.n_rows):
        s = 0.0
        for k in range(rp[i], rp[i + 1]):
            s = s + v[k] * x[ci[k]]
        y[i] = s
    return y


def test_residual_fused(H, orc):
    import torch
    for a in matrices(H)[:5]:
        rng = np.random.default_rng(3)
        x, b = rng.uniform(-1, 1, a.n_cols), rng.uniform(-1, 1, a.n_rows)
        sp = H.DeviceSpmv(a)
        xd, bd = torch.tensor(x, device="cuda"), torch.tensor(b, device="cuda")
        y = torch.empty_like(bd)
        sp.residual(bd, xd, y)
        torch.cuda.synchronize()
        assert bits_equal(y.cpu().numpy(), b - orc.spmv(to_oracle(a), x))


def test_golden_b(H):
    d = load("poisson_ilu")  # b = A*1 produced by the reference's spmv_csr
    assert bits_equal(H.spmv_csr(H.gen_poisson7(12, 10, 8), np.ones(960)), d["b"])


def test_empty(H):
    a = H.csr_from_triples(0, 0, [])
    assert H.spmv_csr(a, np.zeros(0)).shape == (0,)


def test_poisson_256_bitwise(H, orc):
    a = H.gen_poisson7(256, 256, 256)
    x = np.random.default_rng(4).uniform(-1, 1, a.n_cols)
    assert bits_equal(H.DeviceSpmv(a).run_host(x), orc.spmv(to_oracle(a), x))
