"""Bitwise parity at the BASELINE.json config sizes (SURVEY.md 8(d) C1, C2, C4,
C5), on the device layouts those sizes select.

The device layout is picked by size-dependent branches of the planner
(tri_plan.cpp: z-plane slabs of 128 CTAs for 27-point 128^3, z-pencils with a
1024-entry x ring for 7-point 256^3, strips for RCM orderings, level launches
for random orderings), so small-system tests do not reach them. Pattern of the
reference's acceptance.cpp:152-177 (prepared solve checked against a second
implementation on the same inputs):

* the matrix comes from the C oracle's generators (oracle/hec_oracle.c), the
  factors and prepared triangles from the REFERENCE itself (oracle/_ref:
  hecref::ilu0 / prepare_lower / prepare_upper); the product's own setup must
  reproduce them exactly at full size;
* every device result -- L solve, U solve, the ILU apply (L's output kept in
  wave order, composed gather into U) and the C-ABI host entry
  hec_precond_apply_host -- must equal hecref::solve bit for bit
  (triangular.cpp:90-135; north_star allows 1e-12, we require 0).
"""
import os

import numpy as np
import pytest

from util import bits_equal

pytestmark = pytest.mark.gpu

CORES = os.cpu_count() or 1

# name: (stencil, edge, ordering, expected device layout: 0 slabs, 1 pencils, 2 strips, None levels)
CASES = {
    "c1_p7_64": (7, 64, "natural", 1),
    "c2_p27_128": (27, 128, "natural", 0),
    "c4_p7_256": (7, 256, "natural", 1),
    "c5_p7_100_rcm": (7, 100, "rcm", 1),  # z-pencils from the DAG's grid coordinates
    "c5_p7_100_random": (7, 100, "random", None),
}


class Case:
    pass


@pytest.fixture(scope="module", params=list(CASES))
def case(request, H, orc, ref):
    from oracle.oracle import Csr
    stencil, s, ordering, layout = CASES[request.param]
    c = Case()
    c.name, c.layout = request.param, layout
    A = orc.poisson7(s, s, s) if stencil == 7 else orc.poisson27(s, s, s)
    a = H.gen_poisson7(s, s, s) if stencil == 7 else H.gen_poisson27(s, s, s)
    assert bits_equal(np.asarray(a.values), A.v) and bits_equal(np.asarray(a.col_indices), A.ci)
    if ordering != "natural":
        perm = H.rcm_ordering(a) if ordering == "rcm" else H.random_ordering(a.n_rows)
        a = H.permute_symmetric(a, perm)
        A = Csr.of(a)
    c.n = A.n
    # the reference's setup (hecref::ilu0, prepare_lower / prepare_upper)
    c.rl, c.ru = ref.ilu(A)
    c.prl, c.pru = ref.prepare(c.rl), ref.prepare(c.ru, upper=True)
    # the product's setup
    f = H.ilu0(a)
    c.f = f
    c.pl, c.pu = H.prepare_lower(f.l), H.prepare_upper(f.u)
    c.b = ref.spmv(A, np.ones(A.n), CORES)  # b = A*1 (bench.cpp:110-111)
    c.br = np.random.default_rng(1606).uniform(-1.0, 1.0, A.n)
    c.y = ref.solve(c.prl, c.b, CORES)
    c.x = ref.solve(c.pru, c.y, CORES)
    c.yr = ref.solve(c.prl, c.br, CORES)
    c.xr = ref.solve(c.pru, c.yr, CORES)
    yield c


def _prep_equal(p, q):
    s, e = p.schedule, p.hec
    return (p.n == q.n and s.nlev == q.nlev and int(p.reversal_applied) == q.reversed
            and bits_equal(np.asarray(s.level_of), q.level_of) and bits_equal(np.asarray(s.perm), q.perm)
            and bits_equal(np.asarray(s.inv_perm), q.inv_perm)
            and bits_equal(np.asarray(s.level_starts), q.level_starts) and e.ell.width == q.width
            and bits_equal(np.asarray(e.ell.col_indices), q.ell_cols)
            and bits_equal(np.asarray(e.ell.values), q.ell_vals)
            and bits_equal(np.asarray(e.csr_row_offsets), q.csr_rp)
            and bits_equal(np.asarray(e.csr_col_indices), q.csr_ci)
            and bits_equal(np.asarray(e.csr_values), q.csr_v))


def test_setup_bitwise_at_size(case):
    from oracle.oracle import Csr
    for mine, theirs in ((case.f.l, case.rl), (case.f.u, case.ru)):
        m = Csr.of(mine)
        assert bits_equal(m.rp, theirs.rp) and bits_equal(m.ci, theirs.ci) and bits_equal(m.v, theirs.v)
    assert _prep_equal(case.pl, case.prl.prepared())
    assert _prep_equal(case.pu, case.pru.prepared())


def _dev(x):
    import torch
    return torch.tensor(x, dtype=torch.float64, device="cuda")


def test_layout_is_the_benchmarked_one(H, case):
    info = H.DeviceTri.create(case.pl).info()
    print(case.name, info)
    if case.layout is None:
        assert info["strategy"] == 1
    else:
        assert info["strategy"] == 2 and info["layout"] == case.layout, info


def test_lower_and_upper_solves_bitwise(H, case):
    import torch
    tl, tu = H.DeviceTri.create(case.pl), H.DeviceTri.create(case.pu)
    for b, y_want, x_want in ((case.b, case.y, case.x), (case.br, case.yr, case.xr)):
        bd, yin = _dev(b), _dev(y_want)
        y, x = torch.empty_like(bd), torch.empty_like(bd)
        tl.solve(bd, y)
        tu.solve(yin, x)
        torch.cuda.synchronize()
        assert bits_equal(y.cpu().numpy(), y_want), "L solve differs from hecref::solve"
        assert bits_equal(x.cpu().numpy(), x_want), "U solve differs from hecref::solve"


def test_ilu_apply_bitwise(H, case):
    import torch
    dp = H.DevicePrecond.create(case.n, case.pl, case.pu)
    for b, x_want in ((case.b, case.x), (case.br, case.xr)):
        bd = _dev(b)
        x = torch.empty_like(bd)
        for _ in range(3):  # repeated applies reuse the mailboxes (epoch tags)
            x.fill_(np.nan)
            dp.apply(bd, x)
            torch.cuda.synchronize()
            assert bits_equal(x.cpu().numpy(), x_want), "device ILU apply differs from hecref"
        assert bits_equal(dp.apply_host(b), x_want), "hec_precond_apply_host differs from hecref"


def test_dropin_solve_bitwise(H, case):
    # hec::solve drop-in (host vectors in and out, the reference's signature)
    assert bits_equal(H.solve(case.pu, H.solve(case.pl, case.br)), case.xr)


# ---------------------------------------------------------------- C3 ----
C3_GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c3_gmres.json")


def _c3_keys():
    import json
    if not os.path.exists(C3_GOLDEN):
        return []
    return sorted(json.load(open(C3_GOLDEN)))


@pytest.mark.parametrize("key", _c3_keys())
def test_c3_gmres_iterations_vs_reference(H, key):
    """BASELINE config C3: reservoir 7-point, one block of ilu0 / ilu_k(1) /
    ilut(10, 1e-3) factors inside GMRES(30), b = A*1, rel_tol 1e-6. Iteration
    counts within +-1 of hecref::gmres (tests/golden/make_c3_golden.py) and the
    solution as close to 1 as the reference's within 2x."""
    import json
    g = json.load(open(C3_GOLDEN))[key]
    s = g["size"]
    a = H.gen_reservoir7(s, s, s)
    b = H.spmv_csr(a, np.ones(a.n_rows), workers=CORES)
    kind = {"ilu0": ("bilu0", {}), "ilu1": ("biluk", {"fill_level": 1}),
            "ilut": ("bilut", {"ilut_p": 10, "ilut_tol": 1e-3})}[g["factor"]]
    m = H.build_preconditioner(a, kind[0], 1, 0, **kind[1])
    res = H.gmres(a, b, m, H.SolverConfig(restart=30, rel_tol=1e-6))
    print(key, res.report.iterations, "reference", g["iterations"])
    assert res.report.converged == g["converged"]
    assert abs(res.report.iterations - g["iterations"]) <= 1, (res.report.iterations, g["iterations"])
    assert res.report.final_relative_residual <= 1e-6
    assert np.max(np.abs(res.x - 1.0)) <= 2.0 * g["max_abs_error_vs_ones"]
