"""The product's host setup (C++ behind the C-ABI) reproduces the reference bit
for bit: prepared schedules / HEC arrays, ILU(0)/ILU(k)/ILUT factors, partitions
and RAS maps (golden fixtures made by the reference, plus live sweeps against
oracle/_ref when built), with the reference's error behaviour. CPU only."""
import numpy as np
import pytest

from golden_util import PREP_FIELDS, csr, load, prepared, product_prepared_arrays, oracle_prepared_arrays
from util import bits_equal, to_oracle, to_product


def same_csr(m, ref):
    return bits_equal(np.asarray(m.row_offsets), ref.rp) and bits_equal(np.asarray(m.col_indices), ref.ci) and \
        bits_equal(np.asarray(m.values), ref.v)


def assert_prepared_equal(p, want, what):
    assert p.n == want.n and p.schedule.nlev == want.nlev and p.hec.ell.width == want.width, what
    assert p.reversal_applied == bool(want.reversed), what
    for f, got, exp in zip(PREP_FIELDS, product_prepared_arrays(p), oracle_prepared_arrays(want)):
        assert bits_equal(np.asarray(got), np.asarray(exp)), (what, f)


def test_golden_random_prepare(H):
    d = load("tri_random")
    for k in range(int(d["count"][0])):
        a = to_product(H, csr(d, f"s{k}_a_"))
        upper = bool(d[f"s{k}_kind"][0])
        p = (H.prepare_upper if upper else H.prepare_lower)(a)
        assert_prepared_equal(p, prepared(d, f"s{k}_p_"), k)
        assert bits_equal((H.serial_backward_solve if upper else H.serial_forward_solve)(a, d[f"s{k}_b"]),
                          d[f"s{k}_x_serial"])


def test_golden_poisson_ilu_and_prepare(H):
    d = load("poisson_ilu")
    a = H.gen_poisson7(12, 10, 8)
    assert same_csr(a, csr(d, "a_"))
    f = H.ilu0(a)
    assert same_csr(f.l, csr(d, "l_")) and same_csr(f.u, csr(d, "u_"))
    assert_prepared_equal(H.prepare_lower(f.l), prepared(d, "pl_"), "L")
    assert_prepared_equal(H.prepare_upper(f.u), prepared(d, "pu_"), "U")
    for w in (0, 1, 5):
        assert_prepared_equal(H.prepare_lower(f.l, H.WidthPolicy.fixed(w)), prepared(d, f"pl_w{w}_"), w)
    # (the product's spmv_csr runs on the device: tests/test_gpu_spmv.py checks it against d["b"])


@pytest.mark.parametrize("name", ["dd", "p7"])
def test_golden_ilu_variants(H, name):
    d = load("ilu_variants")
    a = to_product(H, csr(d, f"{name}_"))
    for tag, fn in (("ilu0", lambda m: H.ilu0(m)), ("iluk1", lambda m: H.ilu_k(m, 1)),
                    ("iluk2", lambda m: H.ilu_k(m, 2)), ("ilut10", lambda m: H.ilut(m, 10, 1e-3)),
                    ("ilut3", lambda m: H.ilut(m, 3, 0.05))):
        f = fn(a)
        assert same_csr(f.l, csr(d, f"{name}_{tag}_l_")), tag
        assert same_csr(f.u, csr(d, f"{name}_{tag}_u_")), tag


def test_golden_preconditioner_maps(H):
    d = load("precond")
    a = to_product(H, csr(d, "a_"))
    for tag, (kind, blocks, overlap) in {"bilu0": ("bilu0", 4, 0), "ras": ("ras", 3, 1),
                                         "bilut": ("bilut", 3, 0)}.items():
        m = H.build_preconditioner(a, kind, blocks, overlap)
        assert bits_equal(m.part_of, d[f"{tag}_part_of"]), tag
        assert bits_equal(m.offsets, d[f"{tag}_offsets"]), tag
        assert bits_equal(m.ext_rows, d[f"{tag}_ext_rows"]), tag
        assert bits_equal(m.owned, d[f"{tag}_owned"]), tag
        assert_prepared_equal(m.prepared_l, prepared(d, f"{tag}_l_"), tag + "L")
        assert_prepared_equal(m.prepared_u, prepared(d, f"{tag}_u_"), tag + "U")


def test_partition_known_answers(H):
    # reference test_partition.cpp:92-148 / test_precond.cpp:122-130
    tri = H.csr_from_triples(4, 4, [(i, j, 2.0 if i == j else -1.0) for i in range(4) for j in range(4)
                                    if abs(i - j) <= 1])
    m = H.build_preconditioner(tri, "ras", 2, 1)
    assert [list(p) for p in m.parts] == [[0, 1], [2, 3]]
    assert [list(p) for p in m.extended_parts] == [[0, 1, 2], [1, 2, 3]]
    assert list(m.offsets) == [0, 3, 6]
    blocks = [(i, j, v) for i, j, v in
              [(0, 0, 5.0), (0, 1, 1.0), (0, 2, 2.0), (1, 0, 1.0), (1, 1, 6.0), (1, 2, -1.0), (2, 0, -2.0),
               (2, 1, 1.0), (2, 2, 7.0)]]
    blocks += [(3 + i, 3 + j, v) for i, j, v in blocks]
    m2 = H.build_preconditioner(H.csr_from_triples(6, 6, blocks), "bilu0", 2, 0)
    assert [list(p) for p in m2.parts] == [[0, 1, 2], [3, 4, 5]]


def test_error_conventions(H):
    # reference test_triangular.cpp:219-230, test_hec.cpp:52-57, test_precond.cpp:176-196
    zero_diag = H.csr_from_triples(2, 2, [(0, 0, 0.0), (1, 1, 1.0)])
    with pytest.raises(H.ZeroPivotError):
        H.prepare_lower(zero_diag)
    with pytest.raises(H.ZeroPivotError):
        H.prepare_upper(zero_diag)
    with pytest.raises(H.ZeroPivotError):
        H.serial_forward_solve(zero_diag, [1.0, 1.0])
    no_diag = H.csr_from_triples(2, 2, [(0, 0, 1.0), (1, 0, 1.0)])
    with pytest.raises(ValueError):
        H.prepare_lower(no_diag)
    with pytest.raises(ValueError):
        H.prepare_lower(H.gen_poisson7(1, 1, 1), H.WidthPolicy.fixed(-1))
    with pytest.raises(IndexError):
        H.csr_from_triples(2, 2, [(2, 0, 1.0)])
    with pytest.raises(ValueError):
        H.csr_from_triples(2, 2, [(0, 0, 1.0), (0, 0, 2.0)])
    tri = H.csr_from_triples(6, 6, [(i, j, 2.0 if i == j else -1.0) for i in range(6) for j in range(6)
                                    if abs(i - j) <= 1])
    with pytest.raises(ValueError):
        H.build_preconditioner(tri, "bilu0", 2, 1)
    with pytest.raises(ValueError):
        H.build_preconditioner(tri, "ras", 2, -1)
    pivots = H.csr_from_triples(4, 4, [(0, 0, 1.0), (1, 1, 1.0), (2, 2, 0.0), (3, 3, 1.0)])
    with pytest.raises(H.ZeroPivotError) as e:
        H.build_preconditioner(pivots, "bilu0", 2, 0)
    assert e.value.block == 1 and e.value.row == 0
    with pytest.raises(ValueError):
        H.ilu_k(tri, -1)
    with pytest.raises(ValueError):
        H.ilut(tri, 0, 0.1)


def test_ilu_k0_equals_ilu0_and_reservoir_reduces(H):
    a = H.gen_reservoir7(9, 8, 7)
    f0, fk = H.ilu0(a), H.ilu_k(a, 0)
    assert f0.l == fk.l and f0.u == fk.u
    # sigma = 0, kz_ratio = 1 is the plain 7-point Poisson operator, bitwise
    assert H.gen_reservoir7(9, 8, 7, 0.0, 1.0) == H.gen_poisson7(9, 8, 7)


def test_poisson27_and_orderings(H):
    a = H.gen_poisson27(5, 4, 3)
    span = lambda d: 3 * d - 2 if d > 1 else 1  # noqa: E731
    assert a.nnz() == span(5) * span(4) * span(3)
    assert H.gen_poisson27(1, 1, 1).values.tolist() == [26.0]
    dense = np.zeros((a.n_rows, a.n_rows))
    for i in range(a.n_rows):
        dense[i, a.col_indices[a.row_offsets[i]:a.row_offsets[i + 1]]] = a.values[a.row_offsets[i]:a.row_offsets[i + 1]]
    assert (dense == dense.T).all() and (np.diag(dense) == 26.0).all()
    p = H.random_ordering(a.n_rows, 1606)
    assert sorted(p.tolist()) == list(range(a.n_rows))
    b = H.permute_symmetric(a, p)
    assert b.nnz() == a.nnz()
    q = H.rcm_ordering(b)
    assert sorted(q.tolist()) == list(range(a.n_rows))
    c = H.permute_symmetric(b, q)

    def bandwidth(m):
        return max(abs(i - j) for i in range(m.n_rows)
                   for j in m.col_indices[m.row_offsets[i]:m.row_offsets[i + 1]])
    assert bandwidth(c) < bandwidth(b)


def test_live_sweep_against_reference(H, ref):
    # acceptance.cpp criteria 2/4/9 style: the product's setup == the reference's
    rng = ref.rng(404)
    for rep in range(30):
        n = rng.uniform_int(20, 400)
        dens = rng.uniform_real(0.01, 0.3)
        kind = ("lower", "upper")[rep % 2]
        t = rng.matrix(kind, n, dens)
        p = (H.prepare_upper if kind == "upper" else H.prepare_lower)(to_product(H, t))
        assert_prepared_equal(p, ref.prepare(t, upper=(kind == "upper")).prepared(), rep)
    for rep in range(10):
        m = rng.matrix("diag_dominant", rng.uniform_int(20, 150), rng.uniform_real(0.02, 0.2))
        pm = to_product(H, m)
        for kind, args, fn in (("ilu0", (), H.ilu0), ("iluk", (2,), H.ilu_k), ("ilut", (5, 0.01), H.ilut)):
            rl, ru = ref.ilu(m, kind, *(args if args else (0,)))
            f = fn(pm, *args)
            assert same_csr(f.l, rl) and same_csr(f.u, ru), (rep, kind)
