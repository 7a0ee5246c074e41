"""GPU parity of the widened path: device SpMV (bitwise vs spmv_csr), the
block-ILU / RAS preconditioner apply (bitwise vs the reference's apply, golden
vectors and the C oracle), and device GMRES (iteration counts within +-1 of the
reference)."""
import numpy as np
import pytest

from golden_util import csr, load, prepared
from util import bits_equal, random_diag_dominant, to_oracle, to_product

pytestmark = pytest.mark.gpu


def test_device_spmv_bitwise(H, orc):
    for a in (H.gen_poisson7(17, 13, 11), H.gen_poisson27(9, 8, 7), H.gen_reservoir7(10, 9, 8)):
        x = np.random.default_rng(1).uniform(-1, 1, a.n_cols)
        got = H.DeviceSpmv(a).run_host(x)
        assert bits_equal(got, orc.spmv(to_oracle(a), x))
        assert bits_equal(got, H.spmv_csr(a, x))


def test_apply_matches_reference_golden(H):
    d = load("precond")
    a = to_product(H, csr(d, "a_"))
    for tag, (kind, blocks, overlap) in {"bilu0": ("bilu0", 4, 0), "ras": ("ras", 3, 1),
                                         "bilut": ("bilut", 3, 0)}.items():
        m = H.build_preconditioner(a, kind, blocks, overlap)
        assert bits_equal(H.apply(m, d["r"]), d[f"{tag}_apply"]), tag


@pytest.mark.parametrize("strategy,long_min", [(1, ""), (1, "1"), (2, "")])  # "1": every remainder a warp row
def test_apply_vs_oracle(H, orc, monkeypatch, strategy, long_min):
    if long_min:
        monkeypatch.setenv("HEC_LEVELS_LONG", long_min)
    rng = np.random.default_rng(61)
    mats = [H.gen_poisson7(14, 12, 10), to_product(H, random_diag_dominant(300, 0.02, rng)),
            H.gen_reservoir7(12, 11, 10)]
    for a in mats:
        for kind, blocks, overlap, extra in (("bilu0", 5, 0, {}), ("ras", 4, 1, {}), ("ras", 3, 2, {}),
                                             ("bilut", 3, 0, {}), ("biluk", 2, 0, {"fill_level": 1})):
            m = H.build_preconditioner(a, kind, blocks, overlap, **extra)
            r = rng.uniform(-1, 1, a.n_rows)
            want = orc.apply(a.n_rows, m.ext_rows, m.owned, to_oracle_prep(orc, m.prepared_l),
                             to_oracle_prep(orc, m.prepared_u), r)
            dp = H.DevicePrecond.create(a.n_rows, m.prepared_l, m.prepared_u, m.ext_rows, m.owned,
                                        strategy=strategy)
            assert bits_equal(dp.apply_host(r), want), (kind, blocks, overlap)


@pytest.mark.parametrize("slices", ["1", "2", "3", "8"])
@pytest.mark.parametrize("dims", [(40, 38, 36), (33, 17, 9), (64, 64, 20)])
def test_apply_host_sliced_copies(H, orc, monkeypatch, slices, dims):
    # hec_precond_apply_host with the host copies cut into slices (each input
    # slice permuted while the next is in flight, each output slice copied back
    # while the next is permuted; default: 2^20 rows a slice, at most 8) gives
    # the unsliced result bit for bit, for row counts that do not divide evenly
    monkeypatch.setenv("HEC_HOST_SLICES", slices)
    a = H.gen_reservoir7(*dims, seed=3)
    f = H.ilu0(a)
    b = np.random.default_rng(17).uniform(-1, 1, a.n_rows)
    y = orc.solve(orc.prepare(to_oracle(f.l)), b)
    want = orc.solve(orc.prepare(to_oracle(f.u), upper=True), y)
    dp = H.DevicePrecond.create(a.n_rows, H.prepare_lower(f.l), H.prepare_upper(f.u))
    for _ in range(2):  # the slice streams and events are reused
        assert bits_equal(dp.apply_host(b), want)


def to_oracle_prep(orc, p):
    from oracle.oracle import Prepared
    s, e = p.schedule, p.hec
    return Prepared(1 if p.kind == "upper" else 0, p.n, int(p.reversal_applied), s.nlev, s.level_of, s.perm,
                    s.inv_perm, s.level_starts, e.ell.width, e.ell.col_indices, e.ell.values, e.csr_row_offsets,
                    e.csr_col_indices, e.csr_values)


def test_collapse_identities(H):
    # reference test_precond.cpp:75-99: ras(overlap 0) == bilu0; single block == global ILU(0) solve
    rng = np.random.default_rng(73)
    a = to_product(H, random_diag_dominant(120, 0.05, rng))
    r = rng.uniform(-1, 1, 120)
    f = H.ilu0(a)
    glob = H.solve(H.prepare_upper(f.u), H.solve(H.prepare_lower(f.l), r))
    assert bits_equal(H.apply(H.build_preconditioner(a, "bilu0", 1, 0), r), glob)
    assert bits_equal(H.apply(H.build_preconditioner(a, "ras", 1, 1), r), glob)
    assert bits_equal(H.apply(H.build_preconditioner(a, "ras", 3, 0), r),
                      H.apply(H.build_preconditioner(a, "bilu0", 3, 0), r))


def test_apply_is_linear_and_blockwise(H):
    # reference test_precond.cpp:148-172
    tri = H.csr_from_triples(10, 10, [(i, j, 2.0 if i == j else -1.0) for i in range(10) for j in range(10)
                                      if abs(i - j) <= 1])
    m = H.build_preconditioner(tri, "ras", 2, 1)
    r = np.ones(10)
    r[m.extended_parts[0]] = 0.0
    x = H.apply(m, r)
    assert (x[m.parts[0]] == 0.0).all()
    rng = np.random.default_rng(97)
    a = to_product(H, random_diag_dominant(80, 0.05, rng))
    m = H.build_preconditioner(a, "ras", 3, 1)
    r1, r2 = rng.uniform(-1, 1, 80), rng.uniform(-1, 1, 80)
    assert np.max(np.abs(H.apply(m, r1 + r2) - H.apply(m, r1) - H.apply(m, r2))) <= 1e-12


def test_gmres_golden_iterations(H):
    d = load("gmres")
    a = to_product(H, csr(d, "a_"))
    b = H.spmv_csr(a, np.ones(a.n_rows))
    for tag, spec in {"none": None, "bilu0": ("bilu0", 4, 0), "ras": ("ras", 4, 1),
                      "bilut": ("bilut", 4, 0)}.items():
        m = H.build_preconditioner(a, *spec) if spec else None
        res = H.gmres(a, b, m, H.SolverConfig(restart=20))
        conv, iters, rel = d[f"{tag}_report"]
        assert res.report.converged == bool(conv), tag
        assert abs(res.report.iterations - int(iters)) <= 1, (tag, res.report.iterations, iters)
        assert res.report.final_relative_residual <= 1e-6
        # the reported residual is the recomputed one (reference gmres.cpp:126-131)
        r = b - H.spmv_csr(a, res.x)
        assert abs(np.linalg.norm(r) / np.linalg.norm(b) - res.report.final_relative_residual) <= 1e-12
        assert np.max(np.abs(res.x - 1.0)) <= 2e-4


def test_gmres_acceptance_40cube(H, ref):
    # reference acceptance.cpp:267-297 (criterion 7): GMRES(20), 16 blocks on 40^3, b = A*1
    a = H.gen_poisson7(40, 40, 40)
    b = H.spmv_csr(a, np.ones(a.n_rows))
    A = to_oracle(a)
    for kind, overlap in (("bilu0", 0), ("ras", 1), ("bilut", 0)):
        m = H.build_preconditioner(a, kind, 16, overlap, 7, 0.1)
        res = H.gmres(a, b, m, H.SolverConfig(restart=20))
        _, rep = ref.gmres(A, b, ref.precond(A, kind, 16, overlap), restart=20)
        assert res.report.converged and res.report.final_relative_residual <= 1e-6
        assert abs(res.report.iterations - rep["iterations"]) <= 1, (kind, res.report.iterations, rep["iterations"])
        assert np.max(np.abs(res.x - 1.0)) <= 1e-4


def test_gmres_edge_cases(H):
    # reference test_gmres.cpp:40-72: identity converges in one step, zero rhs in zero
    eye = H.csr_from_triples(8, 8, [(i, i, 1.0) for i in range(8)])
    b = np.random.default_rng(101).uniform(-1, 1, 8)
    res = H.gmres(eye, b, None, H.SolverConfig())
    assert res.report.converged and res.report.iterations == 1
    assert np.max(np.abs(res.x - b)) <= 1e-14
    tri = H.csr_from_triples(10, 10, [(i, j, 2.0 if i == j else -1.0) for i in range(10) for j in range(10)
                                      if abs(i - j) <= 1])
    res = H.gmres(tri, np.zeros(10), None, H.SolverConfig())
    assert res.report.converged and res.report.iterations == 0 and res.report.final_relative_residual == 0.0
    res = H.gmres(tri, np.ones(10), None, H.SolverConfig(restart=2, max_iters=3))
    assert res.report.iterations <= 3
