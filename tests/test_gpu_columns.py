"""The column-state kernel (k_cols, csrc/cuda/cols_kernel.cu; layout: tri_plan.hpp
COLUMNS) for 7-point grid factors: bitwise equal to the reference's solve
(proj/src/triangular.cpp:90-135, restated by the C oracle) for L, U and the
ILU apply with U as the exact mirror of L, over grid shapes that exercise
partial tiles, every CTA tiling (HEC_COLS_WARPS), warp and CTA tile edges,
special values, CUDA-graph replay and concurrent streams.
"""
import numpy as np
import pytest

from util import bits_equal, to_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _columns_on(monkeypatch):
    monkeypatch.setenv("HEC_WAVE_COLUMNS", "1")

GRIDS = [(28, 26, 24), (33, 17, 9), (8, 4, 130), (41, 37, 5)]


def _factors(H, dims, seed=0):
    # seed: the heterogeneous 7-point reservoir (C3), non-constant factor values
    a = H.gen_reservoir7(*dims, seed=seed) if seed else H.gen_poisson7(*dims)
    return a, H.ilu0(a)


def _want(orc, f, b):
    y = orc.solve(orc.prepare(to_oracle(f.l)), b)
    return y, orc.solve(orc.prepare(to_oracle(f.u), upper=True), y)


@pytest.mark.parametrize("shape", ["", "16x1", "8x2", "4x4", "4x1", "1x4"])  # warps x columns per lane
@pytest.mark.parametrize("dims", GRIDS)
def test_columns_bitwise(H, orc, monkeypatch, dims, shape):
    warps = shape.split("x")[0] if shape else ""
    if shape:
        monkeypatch.setenv("HEC_COLS_WARPS", warps)
        monkeypatch.setenv("HEC_COLS_RPL", shape.split("x")[1])
    a, f = _factors(H, dims, seed=7)
    rng = np.random.default_rng(11)
    b = rng.uniform(-1, 1, a.n_rows)
    y_want, x_want = _want(orc, f, b)
    tl, tu = H.DeviceTri.create(H.prepare_lower(f.l)), H.DeviceTri.create(H.prepare_upper(f.u))
    il, iu = tl.info(), tu.info()
    assert il["layout"] == 4 and iu["layout"] == 4, (il, iu)
    if shape:
        assert (il["group"], il["rows_per_lane"]) == tuple(int(v) for v in shape.split("x")), il
    assert il["wave_len"] >= a.n_rows
    assert bits_equal(tl.solve_host(b), y_want), "L"
    assert bits_equal(tu.solve_host(y_want), x_want), "U"
    dp = H.DevicePrecond.create(a.n_rows, H.prepare_lower(f.l), H.prepare_upper(f.u))
    pl, pu = dp.info()
    assert pl["layout"] == 4 and pu["layout"] == 5, (pl, pu)  # U reads L's output reversed, no gather
    assert bits_equal(dp.apply_host(b), x_want), "apply"


def test_columns_special_values(H, orc):
    # Inf / NaN / signed zeros propagate exactly as in the reference (a missing
    # neighbour contributes nothing, even next to an Inf)
    a, f = _factors(H, (20, 18, 16))
    n = a.n_rows
    rng = np.random.default_rng(3)
    b = rng.uniform(-1, 1, n)
    b[rng.integers(0, n, 5)] = np.inf
    b[rng.integers(0, n, 5)] = -np.inf
    b[rng.integers(0, n, 5)] = np.nan
    b[rng.integers(0, n, 50)] = -0.0
    y_want, x_want = _want(orc, f, b)
    tl = H.DeviceTri.create(H.prepare_lower(f.l))
    assert tl.info()["layout"] == 4
    y = tl.solve_host(b)
    _same(y, y_want)
    dp = H.DevicePrecond.create(n, H.prepare_lower(f.l), H.prepare_upper(f.u))
    _same(dp.apply_host(b), x_want)


def _same(got, want):
    # bitwise, except that a NaN made here by inf - inf is the device's default
    # NaN rather than x86's (any NaN matches any NaN; NaNs from b propagate bitwise)
    nan = np.isnan(want)
    assert (np.isnan(got) == nan).all()
    assert bits_equal(got[~nan], want[~nan])
    assert (np.signbit(got[~nan]) == np.signbit(want[~nan])).all()


def test_columns_decline(H):
    # not a 7-point grid factor (27-point, RCM order), or turned off: other layouts
    a27 = H.gen_poisson27(18, 17, 16)
    assert H.DeviceTri.create(H.prepare_lower(H.ilu0(a27).l)).info()["layout"] != 4
    a = H.gen_poisson7(24, 22, 20)
    ar = H.permute_symmetric(a, H.rcm_ordering(a))
    assert H.DeviceTri.create(H.prepare_lower(H.ilu0(ar).l)).info()["layout"] != 4
    ilu1 = H.ilu_k(a, 1)  # fill beyond the three neighbours
    assert H.DeviceTri.create(H.prepare_lower(ilu1.l)).info()["layout"] != 4


def test_columns_off_switch(H, monkeypatch):
    monkeypatch.setenv("HEC_WAVE_COLUMNS", "0")
    a = H.gen_poisson7(28, 26, 24)
    assert H.DeviceTri.create(H.prepare_lower(H.ilu0(a).l)).info()["layout"] == 1  # z-pencils


def test_columns_graph_replay_and_streams(H, orc):
    # mailbox epochs advance on the device: captured solves replay bitwise; two
    # streams use separate workspaces
    torch = pytest.importorskip("torch")
    a, f = _factors(H, (30, 28, 26), seed=5)
    dp = H.DevicePrecond.create(a.n_rows, H.prepare_lower(f.l), H.prepare_upper(f.u))
    rng = np.random.default_rng(9)
    bs = [rng.uniform(-1, 1, a.n_rows) for _ in range(3)]
    wants = [_want(orc, f, b)[1] for b in bs]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    bd = torch.tensor(bs[0], device="cuda")
    x1, x2 = torch.empty_like(bd), torch.empty_like(bd)
    b2 = torch.tensor(bs[1], device="cuda")
    with torch.cuda.stream(s1):
        dp.apply(bd, x1, s1)  # first use of the stream outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s1):
        dp.apply(bd, x1, s1)
    for k in range(3):
        bd.copy_(torch.tensor(bs[k], device="cuda"))
        g.replay()
        with torch.cuda.stream(s2):
            dp.apply(b2, x2, s2)
        torch.cuda.synchronize()
        assert bits_equal(x1.cpu().numpy(), wants[k]), k
        assert bits_equal(x2.cpu().numpy(), wants[1])
