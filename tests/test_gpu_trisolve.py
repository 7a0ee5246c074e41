"""GPU parity of the triangular solve (the hot path) against the oracle.

Bar: bitwise equality with the reference's Algorithm 2 (reference
triangular.cpp:90-135) as restated in oracle/hec_oracle.c, for both device
strategies; <= 1e-12 relative to serial substitution (the reference's own
tolerance, test_triangular.cpp:232-254). All calls go through the C-ABI.
"""
import numpy as np
import pytest

from util import bits_equal, random_triangular, rel_inf_error, to_oracle, to_product

pytestmark = pytest.mark.gpu

STRATS = [1, 2]  # HEC_STRATEGY_LEVELS, HEC_STRATEGY_PIPELINE


def device_solve(H, p, b, strategy, ctas=0):
    t = H.DeviceTri.create(p, strategy=strategy, ctas=ctas)
    return t.solve_host(b), t.info()


@pytest.mark.parametrize("strategy", STRATS)
def test_hand_systems(H, strategy):
    # reference test_triangular.cpp:150-173
    l3 = H.csr_from_triples(3, 3, [(0, 0, 2.0), (1, 0, 1.0), (1, 1, 3.0), (2, 1, 2.0), (2, 2, 4.0)])
    x, _ = device_solve(H, H.prepare_lower(l3), np.array([2.0, 4.0, 6.0]), strategy)
    assert x.tolist() == [1.0, 1.0, 1.0]
    u2 = H.csr_from_triples(2, 2, [(0, 0, 2.0), (0, 1, 1.0), (1, 1, 4.0)])
    x, _ = device_solve(H, H.prepare_upper(u2), np.array([3.0, 4.0]), strategy)
    assert x.tolist() == [1.0, 1.0]
    eye = H.csr_from_triples(3, 3, [(0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0)])
    b = np.array([5.0, -2.0, 0.5])
    for prep in (H.prepare_lower, H.prepare_upper):
        x, _ = device_solve(H, prep(eye), b, strategy)
        assert bits_equal(x, b)


def test_dropin_solve_api(H):
    l3 = H.csr_from_triples(3, 3, [(0, 0, 2.0), (1, 0, 1.0), (1, 1, 3.0), (2, 1, 2.0), (2, 2, 4.0)])
    p = H.prepare_lower(l3)
    assert H.solve(p, [2.0, 4.0, 6.0]).tolist() == [1.0, 1.0, 1.0]
    with pytest.raises(ValueError):
        H.solve(p, [1.0, 2.0])


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("upper", [False, True])
def test_random_systems_bitwise(H, orc, strategy, upper):
    rng = np.random.default_rng(101 if not upper else 103)
    for rep in range(25):
        n = int(rng.integers(1, 400))
        dens = float(rng.uniform(0.005, 0.3))
        t = random_triangular(n, dens, rng, upper=upper)
        b = rng.uniform(-1, 1, n)
        p = (H.prepare_upper if upper else H.prepare_lower)(to_product(H, t))
        want = orc.solve(orc.prepare(t, upper=upper), b)
        got, _ = device_solve(H, p, b, strategy, ctas=int(rng.integers(1, 9)) if strategy == 2 else 0)
        assert bits_equal(got, want), (rep, n)
        serial = orc.backward(t, b) if upper else orc.forward(t, b)
        assert rel_inf_error(got, serial) <= 1e-12


@pytest.mark.parametrize("strategy", STRATS)
def test_width_policy_invariance(H, strategy):
    # reference test_triangular.cpp:271-281: ELL width never changes the result
    rng = np.random.default_rng(109)
    t = to_product(H, random_triangular(300, 0.1, rng))
    b = rng.uniform(-1, 1, 300)
    base, _ = device_solve(H, H.prepare_lower(t, H.WidthPolicy.fixed(0)), b, strategy)
    for pol in (None, H.WidthPolicy.fixed(2), H.WidthPolicy.fixed(64)):
        x, _ = device_solve(H, H.prepare_lower(t, pol), b, strategy)
        assert bits_equal(x, base)


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("gen,dims", [("gen_poisson7", (24, 20, 16)), ("gen_poisson27", (16, 14, 12)),
                                       ("gen_reservoir7", (20, 18, 16))])
def test_ilu0_factors_bitwise(H, orc, strategy, gen, dims):
    a = getattr(H, gen)(*dims)
    f = H.ilu0(a)
    rng = np.random.default_rng(7)
    b = rng.uniform(-1, 1, a.n_rows)
    for fac, upper in ((f.l, False), (f.u, True)):
        p = (H.prepare_upper if upper else H.prepare_lower)(fac)
        want = orc.solve(orc.prepare(to_oracle(fac), upper=upper), b)
        got, info = device_solve(H, p, b, strategy)
        assert bits_equal(got, want)
        assert info["strategy"] == strategy


@pytest.mark.parametrize("ctas", [1, 3, 37, 148, 296])
def test_pipeline_cta_counts(H, orc, ctas):
    a = H.gen_poisson7(18, 17, 16)
    f = H.ilu_k(a, 1)
    b = np.random.default_rng(3).uniform(-1, 1, a.n_rows)
    for fac, upper in ((f.l, False), (f.u, True)):
        p = (H.prepare_upper if upper else H.prepare_lower)(fac)
        want = orc.solve(orc.prepare(to_oracle(fac), upper=upper), b)
        got, info = device_solve(H, p, b, 2, ctas=ctas)
        assert bits_equal(got, want)


def test_ilut_long_rows(H, orc):
    # ILUT(p=40) rows exceed the sliced width cap (32) -> tail section
    a = H.gen_reservoir7(12, 12, 10)
    f = H.ilut(a, 40, 0.0)
    b = np.random.default_rng(5).uniform(-1, 1, a.n_rows)
    for fac, upper in ((f.l, False), (f.u, True)):
        p = (H.prepare_upper if upper else H.prepare_lower)(fac)
        want = orc.solve(orc.prepare(to_oracle(fac), upper=upper), b)
        for strategy in STRATS:
            got, _ = device_solve(H, p, b, strategy)
            assert bits_equal(got, want)


def _arrow_factor(n, long_every, long_len, rng, upper=False):
    # three bands of rows; band 1 and 2 rows depend on 3 rows of the band before,
    # every long_every-th row on long_len rows of the earlier bands (and one row
    # whose remainder is not a multiple of the warp width)
    band, rows = n // 3, []
    for i in range(n):
        k = min(i // band, 2)
        if k == 0:
            cols = np.zeros(0, int)
        else:
            m = long_len + (i % 7) if i % long_every == 0 else 3
            pool = k * band if m > 3 else band
            cols = np.unique(rng.integers(0, pool, m) + (0 if m > 3 else (k - 1) * band))
        rows.append((cols, rng.uniform(-1, 1, cols.size) / max(cols.size, 1)))
    from util import _csr_from_rows
    full = [(np.append(c, i), np.append(v, 1.5 + rng.uniform())) for i, (c, v) in enumerate(rows)]
    a = _csr_from_rows(n, full)
    if not upper:
        return a
    # the mirror image is upper triangular: row i -> n-1-i
    mir = [(n - 1 - c[::-1], v[::-1]) for c, v in full[::-1]]
    return _csr_from_rows(n, mir)


@pytest.mark.parametrize("long_min", ["", "0", "1", "200"])
@pytest.mark.parametrize("upper", [False, True])
def test_warp_rows_bitwise(H, orc, monkeypatch, long_min, upper):
    # level launches: rows with long CSR remainders solved a warp each (products
    # in parallel, differences in stored order) equal the thread-serial loop of
    # the reference bit for bit; HEC_LEVELS_LONG moves the threshold (0 = off)
    if long_min:
        monkeypatch.setenv("HEC_LEVELS_LONG", long_min)
    rng = np.random.default_rng(211 + upper)
    t = _arrow_factor(6000, 37, 700, rng, upper)
    p = (H.prepare_upper if upper else H.prepare_lower)(to_product(H, t))
    b = rng.uniform(-1, 1, t.n_rows)
    b[::97] = -0.0
    want = orc.solve(orc.prepare(t, upper=upper), b)
    got, info = device_solve(H, p, b, 1)
    assert info["strategy"] == 1
    assert bits_equal(got, want)
    monkeypatch.setenv("HEC_LEVELS_PERSIST", "1")  # one cooperative launch, grid barrier per level
    got, _ = device_solve(H, p, b, 1)
    assert bits_equal(got, want)


def test_warp_rows_at_size(H, orc):
    # 300k rows in three bands, every 256th row of bands 1-2 with ~4000 entries:
    # the level launches' warp rows at a size where every level spans all SMs
    rng = np.random.default_rng(5)
    n, band = 300000, 100000
    cols, rp = [], [0]
    for i in range(n):
        k = i // band
        if k == 0:
            c = np.zeros(0, np.int64)
        elif i % 256 == 0:
            c = np.unique(rng.integers(0, k * band, 4000))
        else:
            c = np.unique(rng.integers((k - 1) * band, k * band, 3))
        cols.append(c)
        cols.append(np.array([i]))
        rp.append(rp[-1] + c.size + 1)
    ci = np.concatenate(cols).astype(np.int32)
    v = rng.uniform(-1, 1, ci.size) / 64.0
    v[np.array(rp[1:]) - 1] = 1.5  # diagonals
    from oracle.oracle import Csr
    t = Csr(n, n, np.array(rp, np.int32), ci, v)
    p = H.prepare_lower(to_product(H, t))
    b = rng.uniform(-1, 1, n)
    got, info = device_solve(H, p, b, 1)
    assert info["strategy"] == 1
    assert bits_equal(got, orc.solve(orc.prepare(t), b))


def test_repeated_and_device_pointer_solves(H, orc):
    torch = pytest.importorskip("torch")
    a = H.gen_poisson7(32, 32, 32)
    f = H.ilu0(a)
    p = H.prepare_lower(f.l)
    t = H.DeviceTri.create(p, strategy=2)
    rng = np.random.default_rng(11)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for rep in range(4):
        b = rng.uniform(-1, 1, a.n_rows)
        want = orc.solve(orc.prepare(to_oracle(f.l)), b)
        bd = torch.tensor(b, device="cuda")
        x1 = torch.empty_like(bd)
        x2 = torch.empty_like(bd)
        torch.cuda.synchronize()
        t.solve(bd, x1, stream=s1)   # concurrent solves on two streams
        t.solve(bd, x2, stream=s2)
        torch.cuda.synchronize()
        assert bits_equal(x1.cpu().numpy(), want)
        assert bits_equal(x2.cpu().numpy(), want)


def test_nonfinite_propagation(H, orc):
    # NaN / Inf in b flow through exactly as in the reference
    a = H.gen_poisson7(8, 8, 8)
    f = H.ilu0(a)
    b = np.ones(a.n_rows)
    b[5] = np.nan
    b[100] = np.inf
    for fac, upper in ((f.l, False), (f.u, True)):
        p = (H.prepare_upper if upper else H.prepare_lower)(fac)
        want = orc.solve(orc.prepare(to_oracle(fac), upper=upper), b)
        for strategy in STRATS:
            got, _ = device_solve(H, p, b, strategy)
            assert bits_equal(got, want)


def test_empty_and_single(H):
    one = H.csr_from_triples(1, 1, [(0, 0, 4.0)])
    for strategy in STRATS:
        x, _ = device_solve(H, H.prepare_lower(one), np.array([2.0]), strategy)
        assert x.tolist() == [0.5]
    empty = H.CsrMatrix.from_arrays(0, 0, np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0))
    p = H.prepare_lower(empty)
    assert H.solve(p, np.zeros(0)).shape == (0,)


@pytest.mark.parametrize("strategy", STRATS)
def test_permute_in_then_ordered_solve(H, orc, strategy):
    # hec_tri_permute_in + hec_tri_solve_ordered == hec_tri_solve, bitwise
    torch = pytest.importorskip("torch")
    for gen, dims in (("gen_poisson7", (20, 17, 9)), ("gen_poisson27", (9, 8, 7))):
        a = getattr(H, gen)(*dims)
        f = H.ilu0(a)
        rng = np.random.default_rng(17)
        for fac, upper in ((f.l, False), (f.u, True)):
            p = (H.prepare_upper if upper else H.prepare_lower)(fac)
            t = H.DeviceTri.create(p, strategy=strategy)
            b = rng.uniform(-1, 1, a.n_rows)
            want = orc.solve(orc.prepare(to_oracle(fac), upper=upper), b)
            bd = torch.tensor(b, device="cuda")
            bp = torch.full((t.info()["wave_len"] + 2,), float("nan"), dtype=torch.float64, device="cuda")
            x = torch.empty_like(bd)
            t.permute_in(bd, bp)
            t.solve_ordered(bp, x)
            torch.cuda.synchronize()
            assert bits_equal(x.cpu().numpy(), want)


def test_wave_width_classes_and_splits(H, orc):
    # every supported sliced-ELL width (1-8, 10, 13, 16) plus CSR tails, and
    # chunks split at 32 rows per warp: ILU(k) / ILUT factors of a 27-point matrix
    a = H.gen_poisson27(12, 11, 10)
    rng = np.random.default_rng(5)
    for fac in (H.ilu_k(a, 1), H.ilut(a, 20, 1e-4), H.ilut(a, 3, 1e-2)):
        for t, upper in ((fac.l, False), (fac.u, True)):
            for w in (1, 2, 3, 4, 5, 7, 8, 11, 16, 40):
                p = (H.prepare_upper if upper else H.prepare_lower)(t, H.WidthPolicy.fixed(w))
                b = rng.uniform(-1, 1, a.n_rows)
                want = orc.solve(orc.prepare(to_oracle(t), upper=upper), b)
                got, info = device_solve(H, p, b, 2, ctas=int(rng.integers(1, 40)))
                assert info["strategy"] == 2
                assert bits_equal(got, want), (w, upper)


@pytest.mark.parametrize("knobs", [{}, {"HEC_WAVE_SLABS": "1"},
                                   {"HEC_WAVE_INFLIGHT": "4"},  # the planner keeps >= 2 slots per group
                                   {"HEC_WAVE_G": "1", "HEC_WAVE_K": "4", "HEC_WAVE_RPL": "2"},
                                   {"HEC_WAVE_G": "2", "HEC_WAVE_K": "4", "HEC_WAVE_RPL": "2"},
                                   {"HEC_WAVE_G": "2", "HEC_WAVE_K": "4", "HEC_WAVE_RPL": "1"},
                                   {"HEC_WAVE_G": "4", "HEC_WAVE_K": "4", "HEC_WAVE_RPL": "1"},
                                   {"HEC_WAVE_G": "4", "HEC_WAVE_K": "2", "HEC_WAVE_RPL": "4"},
                                   {"HEC_WAVE_G": "8", "HEC_WAVE_K": "2", "HEC_WAVE_RPL": "2"},
                                   {"HEC_WAVE_G": "4", "HEC_WAVE_K": "3", "HEC_WAVE_RPL": "4"}])
def test_wave_layouts_bitwise(H, orc, knobs, monkeypatch):
    # every row-ownership layout (z-pencils, slabs, strips) and solver shape
    # (G warps per chunk x K groups x RPL rows per lane) gives the reference's bits
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(23)
    cases = [("natural 7pt", H.gen_poisson7(28, 26, 24), None),          # pencils
             ("natural 27pt", H.gen_poisson27(18, 17, 16), None),       # slabs, 1 warp
             ("rcm 7pt", H.gen_poisson7(24, 22, 20), "rcm"),            # pencils (grid from the DAG)
             ("rcm 27pt", H.gen_poisson27(16, 15, 14), "rcm"),          # not pencils
             ("random 7pt", H.gen_poisson7(20, 18, 16), "random")]      # slabs
    for name, a, order in cases:
        if knobs.get("HEC_WAVE_K") == "3" or knobs.get("HEC_WAVE_G") == "8":
            if "27pt" in name:
                continue  # the 8x2x2 and three-group shapes exist for ELL widths <= 4 only
        if order == "rcm":
            a = H.permute_symmetric(a, H.rcm_ordering(a))
        elif order == "random":
            a = H.permute_symmetric(a, H.random_ordering(a.n_rows, 1606))
        f = H.ilu0(a)
        for fac, upper in ((f.l, False), (f.u, True)):
            p = (H.prepare_upper if upper else H.prepare_lower)(fac)
            b = rng.uniform(-1, 1, a.n_rows)
            want = orc.solve(orc.prepare(to_oracle(fac), upper=upper), b)
            got, info = device_solve(H, p, b, 2)
            assert info["strategy"] == 2, name
            assert bits_equal(got, want), (name, upper, knobs)


def test_renumbered_grid_layouts(H, orc):
    # an RCM-renumbered 7-point grid keeps the grid's dependency DAG: the planner
    # recovers the coordinates from it and lays the factor out as z-pencils; a
    # 27-point one (more than three predecessors) does not
    rng = np.random.default_rng(31)
    for a, pencils in ((H.gen_poisson7(26, 24, 22), True), (H.gen_poisson27(16, 15, 14), False)):
        a = H.permute_symmetric(a, H.rcm_ordering(a))
        f = H.ilu0(a)
        for fac, upper in ((f.l, False), (f.u, True)):
            p = (H.prepare_upper if upper else H.prepare_lower)(fac)
            b = rng.uniform(-1, 1, a.n_rows)
            want = orc.solve(orc.prepare(to_oracle(fac), upper=upper), b)
            got, info = device_solve(H, p, b, 2)
            assert (info["layout"] == 1) == pencils, info
            assert bits_equal(got, want)


def test_cuda_graph_replay(H, orc):
    # the mailbox epoch lives on the device (advanced by the kernel), so an
    # L+U pair captured once in a CUDA graph replays with the reference's bits
    torch = pytest.importorskip("torch")
    a = H.gen_poisson7(30, 28, 26)
    f = H.ilu0(a)
    tl = H.DeviceTri.create(H.prepare_lower(f.l), strategy=2)
    tu = H.DeviceTri.create(H.prepare_upper(f.u), strategy=2)
    ol, ou = orc.prepare(to_oracle(f.l)), orc.prepare(to_oracle(f.u), upper=True)
    s = torch.cuda.Stream()
    bd = torch.zeros(a.n_rows, dtype=torch.float64, device="cuda")
    y, x = torch.empty_like(bd), torch.empty_like(bd)
    with torch.cuda.stream(s):
        tl.solve(bd, y, stream=s)      # per-stream workspace allocated outside capture
        tu.solve(y, x, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        tl.solve(bd, y, stream=s)
        tu.solve(y, x, stream=s)
    rng = np.random.default_rng(29)
    for rep in range(5):
        b = rng.uniform(-1, 1, a.n_rows)
        bd.copy_(torch.from_numpy(b))
        g.replay()
        torch.cuda.synchronize()
        assert bits_equal(x.cpu().numpy(), orc.solve(ou, orc.solve(ol, b))), rep


def test_cuda_graph_capture_on_a_fresh_stream(H, orc):
    # a new handle's first stream takes the preallocated workspace: capture works
    # without a warm-up solve on that stream (no allocation, no synchronisation)
    torch = pytest.importorskip("torch")
    a = H.gen_poisson7(24, 22, 20)
    f = H.ilu0(a)
    tl = H.DeviceTri.create(H.prepare_lower(f.l), strategy=2)
    ol = orc.prepare(to_oracle(f.l))
    s = torch.cuda.Stream()
    bd = torch.zeros(a.n_rows, dtype=torch.float64, device="cuda")
    y = torch.empty_like(bd)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        tl.solve(bd, y, stream=s)
    b = np.random.default_rng(31).uniform(-1, 1, a.n_rows)
    bd.copy_(torch.from_numpy(b))
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert bits_equal(y.cpu().numpy(), orc.solve(ol, b))


def test_signed_zero_rhs(H, orc):
    # b = A * 1 leaves exact zeros in the interior (the bench right-hand side);
    # zero numerators take the kernel's a * RN(1/d) shortcut and must keep the
    # IEEE sign of 0 / d, bitwise
    for gen, dims in (("gen_poisson27", (14, 13, 12)), ("gen_poisson7", (22, 21, 20))):
        a = getattr(H, gen)(*dims)
        f = H.ilu0(a)
        b = H.spmv_csr(a, np.ones(a.n_rows))
        rng = np.random.default_rng(31)
        neg = rng.random(a.n_rows) < 0.3
        b[(b == 0) & neg] = -0.0
        for fac, upper in ((f.l, False), (f.u, True)):
            p = (H.prepare_upper if upper else H.prepare_lower)(fac)
            want = orc.solve(orc.prepare(to_oracle(fac), upper=upper), b)
            got, _ = device_solve(H, p, b, 2)
            assert bits_equal(got, want), (gen, upper)
            assert (np.signbit(got) == np.signbit(want)).all()


@pytest.mark.parametrize("strategy", STRATS)
def test_wave_order_output(H, orc, strategy):
    # hec_tri_solve_wave leaves x in wave order; hec_tri_permute_out restores the
    # solution order bitwise; the wave output is a permutation of the solution
    torch = pytest.importorskip("torch")
    a = H.gen_poisson7(19, 18, 17)
    f = H.ilu0(a)
    rng = np.random.default_rng(37)
    for fac, upper in ((f.l, False), (f.u, True)):
        p = (H.prepare_upper if upper else H.prepare_lower)(fac)
        t = H.DeviceTri.create(p, strategy=strategy)
        b = rng.uniform(-1, 1, a.n_rows)
        want = orc.solve(orc.prepare(to_oracle(fac), upper=upper), b)
        bd = torch.tensor(b, device="cuda")
        wl = t.info()["wave_len"]  # n, or more for the column layout (padding slots)
        assert wl >= a.n_rows
        bp = torch.empty(wl + 2, dtype=torch.float64, device="cuda")
        xw = torch.empty(wl, dtype=torch.float64, device="cuda")
        x = torch.full_like(bd, float("nan"))
        t.permute_in(bd, bp)
        t.solve_wave(bp, xw)
        t.permute_out(xw, x)
        torch.cuda.synchronize()
        assert bits_equal(x.cpu().numpy(), want)
        got = xw.cpu().numpy().view(np.uint64)
        if wl == a.n_rows:
            assert np.array_equal(np.sort(got), np.sort(want.view(np.uint64)))
        else:
            assert np.isin(want.view(np.uint64), got).all()


_WATCHDOG_CHILD = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import paper_1606_00541_b200 as H
n = 200000  # bidiagonal: a 200000-level chain, two CTAs (slabs): the second one's waiter
            # polls its first dependency for the ~10-30 ms the first CTA's half takes
a = H.csr_from_triples(n, n, [(i, i, 2.0) for i in range(n)] + [(i, i - 1, -1.0) for i in range(1, n)])
t = H.DeviceTri.create(H.prepare_lower(a), strategy=2, ctas=2)
b = torch.ones(n, dtype=torch.float64, device="cuda")
x = torch.empty_like(b)
try:
    t.solve(b, x)
    torch.cuda.synchronize()
    print("SOLVED", float(x[-1].item()))
except Exception as e:
    print("ERROR", type(e).__name__, str(e)[:200])
"""


def test_watchdog_turns_a_stall_into_an_error():
    # the waiters' mailbox polls are bounded (HEC_WAVE_WATCHDOG_MS): with a 1 ms deadline
    # the second CTA's wait cannot be met in time, the kernel traps and the call fails
    # instead of hanging; with the default deadline the same solve completes
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _WATCHDOG_CHILD.format(root=root)
    env = dict(os.environ, HEC_WAVE_WATCHDOG_MS="1")
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert "ERROR" in p.stdout, p.stdout + p.stderr[-2000:]
    env.pop("HEC_WAVE_WATCHDOG_MS")
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert "SOLVED" in p.stdout, p.stdout + p.stderr[-2000:]
