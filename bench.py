#!/usr/bin/env python
"""Benchmark of the HEC L+U triangular solve on B200 (the BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--secondary c2]
                    [--impl ours|reference] [--ras-size 256] [--ras-ref-size 64]

One step = the ILU(0) apply x = U^-1 L^-1 b of the configured matrix (the L
solve then the U solve), b = A*1 (reference bench.cpp:110-111). Default config:
the north_star target, 7-point Poisson 256^3; the 27-point
128^3 config is reported with the same keys under "secondary". Metric:
effective HBM GB/s = B_alg / time with B_alg = sum over L,U of 12*nnz_T + 20*n
(SURVEY.md 8(d)); ms_per_step is the L+U time.

  value    device-resident b, CUDA events on the launching stream, K steps
  e2e      the C-ABI host entry (hec_precond_apply_host: H2D b, L, U, D2H x)
           with pinned host buffers, same metric
  roofline dominant kernel k_wave: achieved = algorithmic bytes of the L solve
           (12 nnz_L + 20 n) / mean duration of the k_wave launch alone (events
           around hec_tri_solve_wave), peak = measured copy bandwidth
           (MEASURED_PEAKS.json); traffic = ncu dram bytes of that launch
           (profiles/ncu_summary.json)
  cpu_baseline  the reference's own solve (oracle/_ref = /root/reference/proj/src
           compiled by oracle/Makefile; all host threads, and 1 thread) on a
           bounded sample of steps of the same workload; check.bitwise_vs_reference
           compares the device answer with it bit for bit
  --impl reference  the reference's setup + solve on the host cores, on inputs
           from the C oracle's generators (never imports the product)

Multi-GPU (torchrun): the single triangular solve does not shard (SURVEY.md
8(e)), so N ranks run N independent replicas; value = N * B_alg / max-over-
ranks step time ("scaling": "weak"). The RAS half of the metric does shard:
the "ras" object is RAS-ILU(0) GMRES(30) time-to-solution on 7-pt 256^3 with
one subdomain per GPU (halo exchange + dot all-reduces over NCCL), max over
ranks, plus the same at 64^3 beside the reference's hecref::gmres(ras, N blocks).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(stencil=7, size=64, workload="3D 7-point Poisson 64^3, ILU(0), HEC L-solve + U-solve, FP64 (BASELINE config 0)"),
    "c2": dict(stencil=27, size=128, workload="3D 27-point Poisson 128^3, ILU(0) L+U triangular solves, FP64 (BASELINE config 1)"),
    "c4": dict(stencil=7, size=256, workload="3D 7-point Poisson 256^3, ILU(0) L+U triangular solves, FP64 (north_star target)"),
}
PEAK_FALLBACK_GBS = 6650.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return PEAK_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(config_name):
    """dram read+write bytes per k_pipeline launch from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(config_name, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi samples during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 8:
                    continue
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
                for name, v in zip(names, f[4:8]):
                    if v.lower() == "active":
                        reasons.add(name)
        except Exception:
            pass
        finally:
            try:
                os.unlink(self.path)
            except Exception:
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def build_problem(H, cfg):
    t0 = time.time()
    s = cfg["size"]
    a = H.gen_poisson7(s, s, s) if cfg["stencil"] == 7 else H.gen_poisson27(s, s, s)
    b = H.spmv_csr(a, np.ones(a.n_rows), workers=os.cpu_count())
    f = H.ilu0(a)
    pl = H.prepare_lower(f.l)
    pu = H.prepare_upper(f.u)
    log(f"[bench] setup {cfg['stencil']}-pt {s}^3: n={a.n_rows} nnz(L)={f.l.nnz()} nlev={pl.schedule.nlev} "
        f"w={pl.hec.ell.width} in {time.time() - t0:.1f}s")
    return a, b, f, pl, pu


def alg_bytes(p):
    nnz = int(p.hec.csr_row_offsets[-1]) + int(np.count_nonzero(
        p.hec.ell.col_indices.reshape(p.hec.ell.width, p.n) != np.arange(p.n)[None, :])) if p.hec.ell.width else \
        int(p.hec.csr_row_offsets[-1])
    return 12.0 * nnz + 20.0 * p.n


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def measure_config(H, torch, name, args, world, device, with_cpu):
    """One config: device-resident step (value), the dominant kernel alone
    (roofline), the C-ABI host entry with copies (e2e), and on rank 0 at N=1 the
    reference's own solve on the host cores (cpu_baseline, bitwise check)."""
    cfg = CONFIGS[name]
    a, b_host, f, pl, pu = build_problem(H, cfg)
    alg = alg_bytes(pl) + alg_bytes(pu)
    tl = H.DeviceTri.create(pl)
    tu = H.DeviceTri.create(pu)
    dp = H.DevicePrecond.create(pl.n, pl, pu)
    info_l, info_u = tl.info(), tu.info()
    b = torch.tensor(b_host, dtype=torch.float64, device=device)
    y, x, xp = torch.empty_like(b), torch.empty_like(b), torch.empty_like(b)
    stream = torch.cuda.current_stream(device)
    for _ in range(args.warmup):
        dp.apply(b, xp, stream)
        tl.solve(b, y, stream)
        tu.solve(y, x, stream)
    torch.cuda.synchronize(device)
    log(f"[bench] {name}: warm-up done; timing")
    # our kernel launches per step (the ILU apply, DevicePrecond::apply)
    launches = dp.launches_per_apply() if hasattr(dp, "launches_per_apply") else \
        3 + sum(1 if i["strategy"] == 2 else i["nlev"] for i in (info_l, info_u))

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(device)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device.index if device.index is not None else 0) as clocks:
        start.record(stream)
        for _ in range(args.steps):
            dp.apply(b, xp, stream)
        stop.record(stream)
        torch.cuda.synchronize(device)
    total_ms = start.elapsed_time(stop)
    # per triangle (informational): each solve with its own permute-in and permute-out
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    for k in range(args.steps):
        ev[k][0].record(stream)
        tl.solve(b, y, stream)
        ev[k][1].record(stream)
        tu.solve(y, x, stream)
        ev[k][2].record(stream)
    torch.cuda.synchronize(device)
    l_ms = [e[0].elapsed_time(e[1]) for e in ev]
    u_ms = [e[1].elapsed_time(e[2]) for e in ev]
    apply_same = bool((xp.cpu().numpy().view(np.uint64) == x.cpu().numpy().view(np.uint64)).all())
    # the dominant kernel alone: k_wave (L) from an already permuted right-hand side
    wl = info_l["wave_len"]
    bp = torch.empty(wl + 2, dtype=torch.float64, device=device)
    yw = torch.empty(wl, dtype=torch.float64, device=device)
    tl.permute_in(b, bp, stream)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        kev[k][0].record(stream)
        tl.solve_wave(bp, yw, stream)
        kev[k][1].record(stream)
    torch.cuda.synchronize(device)
    wave_ms = [e0.elapsed_time(e1) for e0, e1 in kev]
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
        torch.distributed.barrier()
    ms_step = total_ms / args.steps
    xs = xp.cpu().numpy()
    log(f"[bench] {name}: device step {ms_step:.3f} ms; end-to-end leg")

    # end to end through the C-ABI host entry, pinned buffers, copies inside the timed region
    bh = torch.empty(pl.n, dtype=torch.float64).pin_memory().numpy()
    xh = torch.empty(pl.n, dtype=torch.float64).pin_memory().numpy()
    bh[:] = b_host

    def apply_host():  # the C-ABI call a host application makes (no extra copies)
        H.api.check(H.api.lib.hec_precond_apply_host(dp._h, bh.ctypes.data_as(H.api.L.P_dbl),
                                                     xh.ctypes.data_as(H.api.L.P_dbl)))

    for _ in range(max(1, args.warmup)):
        apply_host()
    e2e_steps = max(3, min(args.steps, 20))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        apply_host()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    e2e_same = bool((xh.view(np.uint64) == xs.view(np.uint64)).all())
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())

    peak, peak_src = measured_peak()
    launch_ms = float(np.mean(wave_ms))
    achieved = alg_bytes(pl) / (launch_ms * 1e-3) / 1e9
    res = {
        "metric": "HEC L+U trisolve effective HBM GB/s (ILU(0) factors, FP64)",
        "value": round(world * alg / (ms_step * 1e-3) / 1e9, 3),
        "unit": "GB/s",
        "ms_per_step": round(ms_step, 4),
        "config": {
            "workload": cfg["workload"], "n": pl.n, "nnz_L": int(f.l.nnz()), "nnz_U": int(f.u.nnz()),
            "nlev_L": int(pl.schedule.nlev), "nlev_U": int(pu.schedule.nlev), "ell_width": int(pl.hec.ell.width),
            "alg_bytes_per_step": alg, "strategy": "pipeline" if info_l["strategy"] == 2 else "levels",
            "layout_L": {0: "slabs", 1: "z-pencils", 2: "strips", 4: "columns"}.get(info_l["layout"], "levels"),
            "solver_shape_L": f"{info_l['group']}x{info_l['groups']}x{info_l['rows_per_lane']}",
            "ctas": info_l["ctas"], "chunks_L": info_l["chunks"], "chunks_U": info_u["chunks"],
            "l2": "inputs larger than L2 (%.0f MB of factors per step vs 126 MB L2)" % (alg / 1e6),
            "parallelism": "replicas" if world > 1 else "single GPU",
        },
        "l_ms": round(float(np.median(l_ms)), 4),
        "u_ms": round(float(np.median(u_ms)), 4),
        "wave_ms_L": round(float(np.median(wave_ms)), 4),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": ncu_traffic(name),
                     "kernel": "k_wave (L solve from a permuted right-hand side)", "peak_source": peak_src,
                     "alg_bytes_per_launch": alg_bytes(pl), "launch_ms": round(launch_ms, 4)},
        "e2e": {"value": round(world * alg / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": 8 * pl.n, "d2h_bytes_per_step": 8 * pl.n,
                "api": "hec_precond_apply_host (C-ABI), pinned host buffers", "bitwise_equal_to_device_path": e2e_same},
        "gpu_launches": int(args.steps * launches),
        "clocks": clocks.summary(),
        "check": {"apply_bitwise_equal_to_separate_solves": apply_same},
    }
    del tl, tu, dp, b, y, x, bp, yw
    if with_cpu:
        med, k, cores, kind, x_ref = cpu_reference_time(pl, pu, b_host, args.cpu_budget, 40)
        w1, k1 = cpu_reference_w1(pl, pu, b_host, args.cpu_budget / 2)
        res["cpu_baseline"] = {
            "value": round(alg / med / 1e9, 4), "unit": "GB/s", "cores": cores, "kind": kind,
            "ms_per_step": round(med * 1e3, 3), "cpu_model": cpu_model(),
            "sample": f"median of {k} full L+U solves of the same workload (hecref::solve, {cores} threads), "
                      f"prepared once from the product's bit-identical setup",
            "w1": {"value": round(alg / w1 / 1e9, 4), "ms_per_step": round(w1 * 1e3, 3), "cores": 1,
                   "sample": f"median of {k1} L+U solves, hecref::solve(.., 1)"}}
        res["check"]["bitwise_vs_reference"] = bool((x_ref.view(np.uint64) == xs.view(np.uint64)).all())
    return res


def _ref_prepared(pl, pu):
    from oracle import load_reference
    ref = load_reference()
    if ref is None:
        raise RuntimeError("oracle/_ref/libhecref.so missing")
    return ref, ref.prepared_from(pl), ref.prepared_from(pu)


def cpu_reference_time(pl, pu, b_host, budget_s, max_steps, min_steps=3):
    """The reference's solve (oracle/_ref), all host threads, on the product's prepared arrays."""
    ref, rl, ru = _ref_prepared(pl, pu)
    cores = os.cpu_count() or 1
    run = lambda b: ref.solve(ru, ref.solve(rl, b, cores), cores)  # noqa: E731
    x = run(b_host)  # warm-up (and the bitwise reference answer)
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < max_steps and (len(times) < min_steps or time.perf_counter() < t_end):
        t0 = time.perf_counter()
        run(b_host)
        times.append(time.perf_counter() - t0)
    return float(np.median(times)), len(times), cores, "reference", x


def cpu_reference_w1(pl, pu, b_host, budget_s, min_steps=2):
    ref, rl, ru = _ref_prepared(pl, pu)
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < min_steps or (time.perf_counter() < t_end and len(times) < 10):
        t0 = time.perf_counter()
        ref.solve(ru, ref.solve(rl, b_host, 1), 1)
        times.append(time.perf_counter() - t0)
    return float(np.median(times)), len(times)


def run_reference_arm(args):
    """--impl reference: the reference's own setup and solve (oracle/_ref, built from
    /root/reference/proj/src) on the host cores. Nothing from the product package:
    the matrix comes from the C oracle's generators."""
    from oracle import load_oracle, load_reference
    cfg = CONFIGS[args.config]
    ref, orc = load_reference(), load_oracle()
    cores = os.cpu_count() or 1
    s = cfg["size"]
    A = orc.poisson7(s, s, s) if cfg["stencil"] == 7 else orc.poisson27(s, s, s)
    if ref is None:
        b = orc.spmv(A, np.ones(A.n))
        l, u = orc.ilu0(A)
        pl, pu = orc.prepare(l), orc.prepare(u, upper=True)
        run = lambda: orc.solve(pu, orc.solve(pl, b))  # noqa: E731
        run1 = run
        kind, cores = "port", 1
        nnz = int(l.rp[-1]) + int(u.rp[-1])
    else:
        b = ref.spmv(A, np.ones(A.n), cores)
        l, u = ref.ilu(A)
        pl, pu = ref.prepare(l), ref.prepare(u, upper=True)
        run = lambda: ref.solve(pu, ref.solve(pl, b, cores), cores)  # noqa: E731
        run1 = lambda: ref.solve(pu, ref.solve(pl, b, 1), 1)  # noqa: E731
        kind = "reference"
        nnz = int(l.rp[-1]) + int(u.rp[-1])
    alg = 12.0 * nnz + 40.0 * A.n
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    ms = float(np.mean(times)) * 1e3
    t1 = []
    for _ in range(2):
        t0 = time.perf_counter()
        run1()
        t1.append(time.perf_counter() - t0)
    ms1 = float(np.median(t1)) * 1e3
    v = round(alg / (ms * 1e-3) / 1e9, 4)
    sample = f"{args.steps} full L+U solves of the {args.config} workload (reference setup excluded)"
    return {
        "metric": "HEC L+U trisolve effective HBM GB/s (ILU(0) factors, FP64)",
        "value": v, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (generated stencil matrix, b = A*1)", "impl": "reference",
        "config": {"workload": cfg["workload"], "n": A.n, "alg_bytes_per_step": alg,
                   "parallelism": "host threads (rank 0 only)"},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": kind, "sample": sample,
                         "cpu_model": cpu_model(),
                         "w1": {"value": round(alg / (ms1 * 1e-3) / 1e9, 4), "ms_per_step": round(ms1, 3),
                                "cores": 1, "sample": "2 L+U solves, hecref::solve(.., 1)"}},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def ras_reference(size, blocks, restart=30):
    """hecref::gmres with build_preconditioner(ras, blocks, overlap 1) on the host
    cores (rank 0): the reference's RAS time-to-solution beside ours."""
    from oracle import load_oracle, load_reference
    ref, orc = load_reference(), load_oracle()
    if ref is None:
        return None
    cores = os.cpu_count() or 1
    A = orc.poisson7(size, size, size)
    b = ref.spmv(A, np.ones(A.n), cores)
    t0 = time.perf_counter()
    m = ref.precond(A, "ras", blocks, 1)
    setup = time.perf_counter() - t0
    x, rep = ref.gmres(A, b, m, restart=restart, rel_tol=1e-6, workers=cores)
    return {"seconds": round(float(rep["solve_seconds"]), 4), "iterations": rep["iterations"],
            "converged": rep["converged"], "setup_seconds": round(setup, 2), "cores": cores,
            "max_abs_error_vs_ones": float(np.max(np.abs(x - 1.0))),
            "what": f"hecref::gmres(restart {restart}) with ras({blocks} blocks, overlap 1), 7-pt {size}^3, "
                    f"{cores} threads"}


def ras_gmres(H, torch, rank, world, device, size, restart=30):
    """RAS-ILU(0) GMRES(restart) time-to-solution, one subdomain per GPU (BASELINE
    config 4), through the library's C++ RAS layer (hec_ras_create / hec_ras_gmres_device:
    NCCL halo exchanges and all-reduces under torchrun). Device-resident b and x,
    CUDA events on the solve's stream, max over ranks."""
    from paper_1606_00541_b200 import ras
    t0 = time.time()
    a = H.gen_poisson7(size, size, size)
    b = H.spmv_csr(a, np.ones(a.n_rows))
    solver = ras.RasSolver(a, overlap=1)
    plan = solver.plan
    setup = time.time() - t0
    log(f"[bench] RAS {size}^3 x{world}: setup {setup:.1f}s ({solver.comm}); warm-up solve")
    bd = torch.tensor(b[plan.own], dtype=torch.float64, device=device)
    xd = torch.empty_like(bd)
    stream = torch.cuda.current_stream(device)
    solver.gmres_device(bd, xd, restart=restart, stream=stream)  # warm-up: layouts, workspaces, NCCL channels
    torch.cuda.synchronize(device)
    if world > 1:
        torch.distributed.barrier()
    # the solve synchronises with the host every iteration (Givens rotations, convergence
    # test), so host-side noise shows: median (and best) of five timed solves
    secs = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rep = solver.gmres_device(bd, xd, restart=restart, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(device)
        secs.append(e0.elapsed_time(e1) * 1e-3)
    err = float((xd - 1.0).abs().max().item())
    if world > 1:  # each solve's time is the slowest rank's
        t = torch.tensor(secs + [err], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        secs, err = [float(v) for v in t[:-1].tolist()], float(t[-1].item())
    sec = float(np.median(secs))
    log(f"[bench] RAS {size}^3 x{world}: {rep.iterations} iterations in {sec*1e3:.1f} ms")
    return {"workload": f"RAS-ILU(0) GMRES({restart}), 7-pt Poisson {size}^3, overlap 1, {world} block(s) = GPU(s), "
                        f"b = A*1, rel_tol 1e-6",
            "seconds": round(sec, 5), "iterations": rep.iterations, "converged": rep.converged,
            "final_relative_residual": rep.final_relative_residual,
            "ms_per_iteration": round(1e3 * sec / max(rep.iterations, 1), 4),
            "max_abs_error_vs_ones": err, "allreduces": rep.allreduces, "halo_exchanges": rep.exchanges,
            "gpu_launches": rep.launches, "rows_per_gpu": plan.n_own, "halo_rows": int(len(plan.halo)),
            "setup_seconds": round(setup, 1), "best_seconds": round(min(secs), 5),
            "seconds_of_solves": [round(v, 5) for v in secs],
            "collectives": ("NCCL all-reduce (2 per iteration, CGS2) + grouped ncclSend/ncclRecv halo exchange"
                            if solver.comm == "nccl" else solver.comm)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--secondary", default="c2", help="second config reported under 'secondary' ('' = none)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of CPU-baseline sampling")
    ap.add_argument("--ras-size", type=int, default=256, help="grid edge of the RAS GMRES run (0 = skip)")
    ap.add_argument("--ras-ref-size", type=int, default=64,
                    help="grid edge of the RAS run timed beside the reference's (0 = skip)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        line = run_reference_arm(args)
        # the reference arm runs the reference library only: the product package must not be loaded
        assert "paper_1606_00541_b200" not in sys.modules, "reference arm imported the product"
        line["product_loaded"] = False
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import paper_1606_00541_b200 as H
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the B200 path has no CPU fallback)")
    device = torch.device("cuda", local % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(device)
    if world > 1:
        # HEC_BENCH_BACKEND=gloo: several ranks on one GPU (control-flow test; RAS then
        # uses host-callback collectives instead of NCCL)
        backend = os.environ.get("HEC_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=device)
        else:
            torch.distributed.init_process_group(backend)
    with_cpu = rank == 0 and world == 1
    head = measure_config(H, torch, args.config, args, world, device, with_cpu)
    result = {"metric": head.pop("metric"), "value": head.pop("value"), "unit": head.pop("unit"), "n_gpus": world,
              "steps": args.steps, "warmup": args.warmup, "ms_per_step": head.pop("ms_per_step"),
              "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
              "data": "synthetic (generated stencil matrix, b = A*1)", "impl": "ours"}
    result.update(head)
    import gc
    gc.collect()
    if args.secondary and args.secondary != args.config:
        result["secondary"] = measure_config(H, torch, args.secondary, args, world, device, with_cpu)
        result["gpu_launches"] += result["secondary"]["gpu_launches"]
        gc.collect()
    if args.ras_size > 0:
        result["ras"] = ras_gmres(H, torch, rank, world, device, args.ras_size)
        if args.ras_ref_size > 0:
            small = ras_gmres(H, torch, rank, world, device, args.ras_ref_size)
            result["ras"]["same_size_as_reference"] = small
            if rank == 0:
                result["ras"]["reference"] = ras_reference(args.ras_ref_size, world)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
