"""Pins the C oracle (oracle/hec_oracle.c) before it is trusted as the checker:
the reference tests' own known answers, the reference-generated golden vectors
in tests/golden/, and (when oracle/_ref is built) fresh random sweeps against
the reference library itself. CPU only."""
import numpy as np
import pytest

from golden_util import PREP_FIELDS, csr, load, oracle_prepared_arrays, prepared
from oracle.oracle import Csr
from util import bits_equal, random_triangular, rel_inf_error

I32 = np.int32


def dense_csr(rows):
    n = len(rows)
    rp, ci, v = [0], [], []
    for i, row in enumerate(rows):
        for j, val in enumerate(row):
            if val != 0.0 or i == j:
                ci.append(j)
                v.append(val)
        rp.append(len(ci))
    return Csr(n, n, np.array(rp, I32), np.array(ci, I32), np.array(v))


def test_hand_triangular(orc):
    # reference test_triangular.cpp:150-173
    l3 = dense_csr([[2, 0, 0], [1, 3, 0], [0, 2, 4]])
    b = np.array([2.0, 4.0, 6.0])
    assert orc.forward(l3, b).tolist() == [1.0, 1.0, 1.0]
    assert orc.solve(orc.prepare(l3), b).tolist() == [1.0, 1.0, 1.0]
    u2 = dense_csr([[2, 1], [0, 4]])
    assert orc.backward(u2, [3.0, 4.0]).tolist() == [1.0, 1.0]
    assert orc.solve(orc.prepare(u2, upper=True), [3.0, 4.0]).tolist() == [1.0, 1.0]


def test_hand_levels_and_schedule(orc):
    # reference test_level_schedule.cpp:23-62 and test_triangular.cpp:186-217
    diag = dense_csr([[1, 0, 0], [0, 1, 0], [0, 0, 1]])
    assert orc.prepare(diag).level_of.tolist() == [1, 1, 1]
    chain = dense_csr([[1, 0, 0], [1, 1, 0], [0, 1, 1]])
    assert orc.prepare(chain).level_of.tolist() == [1, 2, 3]
    fork = dense_csr([[1, 0, 0], [0, 1, 0], [1, 0, 1]])
    p = orc.prepare(fork)
    assert p.level_of.tolist() == [1, 1, 2] and p.perm.tolist() == [0, 1, 2]
    # build_schedule({1,2,1}) -> perm {0,2,1}, starts {0,2,3}
    mid = dense_csr([[1, 0, 0], [1, 1, 0], [0, 0, 1]])
    p = orc.prepare(mid)
    assert p.perm.tolist() == [0, 2, 1] and p.level_starts.tolist() == [0, 2, 3]
    # upper bidiagonal n=5 reverses into a 5-level chain, level_of[i] = i+1
    n = 5
    ub = dense_csr([[2.0 if i == j else (-1.0 if j == i + 1 else 0.0) for j in range(n)] for i in range(n)])
    p = orc.prepare(ub, upper=True)
    assert p.nlev == 5 and p.level_of.tolist() == [1, 2, 3, 4, 5]


def test_hand_hec_layout(orc):
    # reference test_hec.cpp:33-42: bidiagonal, fixed(1)
    bi = dense_csr([[1, 0, 0], [1, 1, 0], [0, 1, 1]])
    p = orc.prepare(bi, fixed_width=1)
    # levels make perm identity here; ELL col {0,0,1}, values {0,1,1}
    assert p.ell_cols.tolist() == [0, 0, 1] and p.ell_vals.tolist() == [0.0, 1.0, 1.0]


def test_hand_ilu_tridiag(orc):
    # reference acceptance.cpp:215-223: tridiag(3) u-diag [2, 1.5, 4/3], l [-0.5, -2/3]
    t = dense_csr([[2, -1, 0], [-1, 2, -1], [0, -1, 2]])
    l, u = orc.ilu0(t)
    # the reference checks these to 1e-14 (acceptance.cpp:224)
    assert np.max(np.abs(np.array([u.v[u.rp[i]] for i in range(3)]) - [2.0, 1.5, 4.0 / 3.0])) <= 1e-14
    assert abs(l.v[l.rp[1]] + 0.5) <= 1e-14 and abs(l.v[l.rp[2]] + 2.0 / 3.0) <= 1e-14


def test_golden_random_systems(orc):
    d = load("tri_random")
    for k in range(int(d["count"][0])):
        a = csr(d, f"s{k}_a_")
        upper = bool(d[f"s{k}_kind"][0])
        want = prepared(d, f"s{k}_p_")
        got = orc.prepare(a, upper=upper)
        for f, ga, wa in zip(PREP_FIELDS, oracle_prepared_arrays(got), oracle_prepared_arrays(want)):
            assert bits_equal(np.asarray(ga), np.asarray(wa)), (k, f)
        x = orc.solve(got, d[f"s{k}_b"])
        assert bits_equal(x, d[f"s{k}_x"]), k
        serial = orc.backward(a, d[f"s{k}_b"]) if upper else orc.forward(a, d[f"s{k}_b"])
        assert bits_equal(serial, d[f"s{k}_x_serial"]), k
        assert rel_inf_error(x, serial) <= 1e-12


def test_golden_poisson(orc):
    d = load("poisson_ilu")
    a = csr(d, "a_")
    assert bits_equal(orc.poisson7(12, 10, 8).v, a.v)
    l, u = orc.ilu0(a)
    for mine, tag in ((l, "l_"), (u, "u_")):
        ref = csr(d, tag)
        assert bits_equal(mine.rp, ref.rp) and bits_equal(mine.ci, ref.ci) and bits_equal(mine.v, ref.v)
    pl, pu = orc.prepare(l), orc.prepare(u, upper=True)
    for got, tag in ((pl, "pl_"), (pu, "pu_")):
        want = prepared(d, tag)
        for f, ga, wa in zip(PREP_FIELDS, oracle_prepared_arrays(got), oracle_prepared_arrays(want)):
            assert bits_equal(np.asarray(ga), np.asarray(wa)), (tag, f)
    assert bits_equal(orc.spmv(a, np.ones(a.n)), d["b"])
    y = orc.solve(pl, d["b"])
    assert bits_equal(y, d["y"])
    assert bits_equal(orc.solve(pu, y), d["x"])
    for w in (0, 1, 5):
        got = orc.prepare(l, fixed_width=w)
        want = prepared(d, f"pl_w{w}_")
        assert got.width == want.width
        assert bits_equal(got.ell_cols, want.ell_cols) and bits_equal(got.csr_v, want.csr_v)
        assert bits_equal(orc.solve(got, d["b"]), d["y"])  # width never changes the result


def test_golden_precond_apply(orc):
    d = load("precond")
    r = d["r"]
    n = len(r)
    for tag in ("bilu0", "ras", "bilut"):
        x = orc.apply(n, d[f"{tag}_ext_rows"], d[f"{tag}_owned"], prepared(d, f"{tag}_l_"),
                      prepared(d, f"{tag}_u_"), r)
        assert bits_equal(x, d[f"{tag}_apply"]), tag


def test_oracle_vs_reference_sweep(orc, ref):
    # acceptance.cpp:123-148 (criterion 2) style sweep against the live reference
    rng = ref.rng(2026)
    for rep in range(40):
        n = rng.uniform_int(10, 600)
        dens = rng.uniform_real(0.005, 0.2)
        kind = "lower" if rep % 2 == 0 else "upper"
        t = rng.matrix(kind, n, dens)
        b = rng.vector(n)
        bag = ref.prepare(t, upper=(kind == "upper"))
        assert bits_equal(orc.solve(orc.prepare(t, upper=(kind == "upper")), b), ref.solve(bag, b, 3))


def test_numpy_generator_systems(orc):
    rng = np.random.default_rng(9)
    for upper in (False, True):
        t = random_triangular(150, 0.1, rng, upper=upper)
        b = rng.uniform(-1, 1, 150)
        x = orc.solve(orc.prepare(t, upper=upper), b)
        serial = orc.backward(t, b) if upper else orc.forward(t, b)
        assert rel_inf_error(x, serial) <= 1e-12
