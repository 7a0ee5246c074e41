#!/usr/bin/env python
"""Benchmark of the HEC L+U triangular solve on B200 (the BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One step = the L solve (b -> y) followed by the U solve (y -> x) of the ILU(0)
factors of the configured matrix, b = A*1 (reference bench.cpp:110-111).
Metric: effective HBM GB/s = B_alg / time with B_alg = sum over L,U of
12*nnz_T + 20*n; ms_per_step is the L+U time.

  value    device-resident b, CUDA events on the launching stream, K steps
  e2e      the C-ABI host entry (hec_precond_apply_host: H2D b, L, U, D2H x)
           with pinned host buffers, same metric
  roofline dominant kernel k_wave: achieved = algorithmic bytes of the L solve
           (12 nnz_L + 20 n) / mean duration of the k_wave launch alone (events
           around hec_tri_solve_ordered), peak = measured copy bandwidth
           (MEASURED_PEAKS.json)
  cpu_baseline  the reference's own solve (oracle/_ref, all host threads) on a
           bounded sample of steps of the same workload

Multi-GPU (torchrun): the single triangular solve does not shard (SURVEY.md
8(e)), so N ranks run N independent replicas; value = N * B_alg / max-over-
ranks step time ("scaling": "weak"). The RAS half of the metric does shard:
the "ras" object is RAS-ILU(0) GMRES(30) time-to-solution on 7-pt 256^3 with
one subdomain per GPU (NCCL halo all-to-all + dot all-reduces), max over ranks.
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


def time_device(H, torch, pl, pu, b_host, steps, warmup, device):
    """Device-resident L+U solve timing; returns per-step ms and per-launch ms.
    The step is the ILU apply x = U^-1 L^-1 b (hec_precond_apply: L's output stays
    in its wave order and U gathers its right-hand side from there)."""
    tl = H.DeviceTri.create(pl)
    tu = H.DeviceTri.create(pu)
    dp = H.DevicePrecond.create(pl.n, pl, pu)
    n = pl.n
    b = torch.tensor(b_host, dtype=torch.float64, device=device)
    y = torch.empty_like(b)
    x = torch.empty_like(b)
    stream = torch.cuda.current_stream(device)
    for _ in range(warmup):
        dp.apply(b, x, stream)
        tl.solve(b, y, stream)
        tu.solve(y, x, stream)
    torch.cuda.synchronize(device)
    time_device.precond = dp
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    return tl, tu, b, y, x, stream, ev, start, stop


def run_ours(args, H, torch, rank, world, device):
    cfg = CONFIGS[args.config]
    a, b_host, f, pl, pu = build_problem(H, cfg)
    alg = alg_bytes(pl) + alg_bytes(pu)
    tl, tu, b, y, x, stream, ev, start, stop = time_device(H, torch, pl, pu, b_host, args.steps, args.warmup, device)
    info_l, info_u = tl.info(), tu.info()
    log("[bench] warm-up done; timing")
    # our kernel launches per step (the ILU apply): permute-in, k_wave L, composed
    # permute, k_wave U, permute-out; one k_level_rows per level with the LEVELS strategy
    launches = 3 + sum(1 if i["strategy"] == 2 else i["nlev"] for i in (info_l, info_u))

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(device)
    dp = time_device.precond
    xp = torch.empty_like(x)
    with ClockSampler(device.index if device.index is not None else 0) as clocks:
        start.record(stream)
        for k in range(args.steps):
            dp.apply(b, xp, stream)
        stop.record(stream)
        torch.cuda.synchronize(device)
    total_ms = start.elapsed_time(stop)
    # per triangle (informational): each solve with its own permute-in and permute-out
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
    # the dominant kernel alone: k_wave from an already permuted right-hand side
    bp = torch.empty(pl.n + 2, dtype=torch.float64, device=device)
    yw = torch.empty_like(y)
    tl.permute_in(b, bp, stream)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        kev[k][0].record(stream)
        tl.solve_wave(bp, yw, stream)
        kev[k][1].record(stream)
    pev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    pev[0].record(stream)
    for k in range(args.steps):
        tl.permute_in(b, bp, stream)
    pev[1].record(stream)
    torch.cuda.synchronize(device)
    wave_ms = [e0.elapsed_time(e1) for e0, e1 in kev]
    permute_ms = pev[0].elapsed_time(pev[1]) / args.steps
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
        torch.distributed.barrier()
    ms_step = total_ms / args.steps

    # correctness guard on the benchmarked output (bitwise vs the oracle at small sizes
    # is in tests/; here: the solve reproduces the all-ones solution of A x = A 1
    # up to ILU(0) being a preconditioner, so check the exact L U x = b residual instead)
    xs = x.cpu().numpy()
    ys = y.cpu().numpy()
    lu_res = float(np.max(np.abs(H.spmv_csr(f.l, ys, workers=os.cpu_count()) - b_host)) /
                   max(1.0, float(np.max(np.abs(b_host)))))
    u_res = float(np.max(np.abs(H.spmv_csr(f.u, xs, workers=os.cpu_count()) - ys)) /
                  max(1.0, float(np.max(np.abs(ys)))))

    log(f"[bench] device step {ms_step:.3f} ms; end-to-end leg")
    # end to end through the C-ABI host entry, pinned buffers, copies inside the timed region
    bh = torch.empty(pl.n, dtype=torch.float64).pin_memory().numpy()
    xh = torch.empty(pl.n, dtype=torch.float64).pin_memory().numpy()
    bh[:] = b_host
    def apply_host():  # the C-ABI call a host application makes (no extra copies)
        H.api.check(H.api.lib.hec_precond_apply_host(dp._h, bh.ctypes.data_as(H.api.L.P_dbl),
                                                     xh.ctypes.data_as(H.api.L.P_dbl)))

    for _ in range(max(1, args.warmup)):
        apply_host()
    t0 = time.perf_counter()
    e2e_steps = max(3, min(args.steps, 20))
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
    result = {
        "metric": "HEC L+U trisolve effective HBM GB/s (ILU(0) factors, FP64)",
        "value": round(world * alg / (ms_step * 1e-3) / 1e9, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (generated stencil matrix, b = A*1)",
        "impl": "ours",
        "config": {
            "workload": cfg["workload"], "n": pl.n, "nnz_L": int(f.l.nnz()), "nnz_U": int(f.u.nnz()),
            "nlev_L": int(pl.schedule.nlev), "nlev_U": int(pu.schedule.nlev), "ell_width": int(pl.hec.ell.width),
            "alg_bytes_per_step": alg, "strategy": "pipeline" if info_l["strategy"] == 2 else "levels",
            "ctas": info_l["ctas"], "chunks_L": info_l["chunks"], "chunks_U": info_u["chunks"],
            "l2": "inputs larger than L2 (%.0f MB of factors per step vs 126 MB L2)" % (alg / 1e6),
            "parallelism": "replicas" if world > 1 else "single GPU",
        },
        "l_ms": round(float(np.median(l_ms)), 4),
        "u_ms": round(float(np.median(u_ms)), 4),
        "wave_ms_L": round(float(np.median(wave_ms)), 4),
        "permute_ms": round(permute_ms, 4),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": ncu_traffic(args.config),
                     "kernel": "k_wave (L solve from a permuted right-hand side)", "peak_source": peak_src},
        "e2e": {"value": round(world * alg / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": 8 * pl.n, "d2h_bytes_per_step": 8 * pl.n,
                "api": "hec_precond_apply_host (C-ABI), pinned host buffers", "bitwise_equal_to_device_path": e2e_same},
        "gpu_launches": int(args.steps * launches),
        "clocks": clocks.summary(),
        "check": {"lu_rel_residual_L": lu_res, "lu_rel_residual_U": u_res,
                  "apply_bitwise_equal_to_separate_solves": apply_same},
    }
    del tl, tu, dp
    return result, (a, b_host, f, pl, pu, alg)


def cpu_reference_time(pl, pu, b_host, budget_s, max_steps, min_steps=3):
    """The reference's solve (oracle/_ref), all host threads, on the product's prepared arrays."""
    from oracle import load_oracle, load_reference
    ref = load_reference()
    cores = os.cpu_count() or 1
    if ref is None:
        raise RuntimeError("oracle/_ref/libhecref.so missing")
    rl, ru = ref.prepared_from(pl), ref.prepared_from(pu)
    run = lambda b: ref.solve(ru, ref.solve(rl, b, cores), cores)  # noqa: E731
    kind = "reference"
    run(b_host)  # warm-up
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < max_steps and (len(times) < min_steps or time.perf_counter() < t_end):
        t0 = time.perf_counter()
        run(b_host)
        times.append(time.perf_counter() - t0)
    return float(np.median(times)), len(times), cores, kind


def cpu_port_time(f, b_host, budget_s, max_steps, min_steps=2):
    """Fallback when the reference .so is absent: the C oracle's Algorithm 2 (1 thread)."""
    from oracle import load_oracle
    from oracle.oracle import Csr
    orc = load_oracle()
    ol, ou = orc.prepare(Csr.of(f.l)), orc.prepare(Csr.of(f.u), upper=True)
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < max_steps and (len(times) < min_steps or time.perf_counter() < t_end):
        t0 = time.perf_counter()
        orc.solve(ou, orc.solve(ol, b_host))
        times.append(time.perf_counter() - t0)
    return float(np.median(times)), len(times), 1, "port"


def run_reference_arm(args):
    """--impl reference: the reference's own setup and solve on the host cores."""
    import paper_1606_00541_b200 as H  # matrix generator only (input data)
    from oracle import load_reference
    from oracle.oracle import Csr
    cfg = CONFIGS[args.config]
    ref = load_reference()
    cores = os.cpu_count() or 1
    s = cfg["size"]
    a = H.gen_poisson7(s, s, s) if cfg["stencil"] == 7 else H.gen_poisson27(s, s, s)
    A = Csr.of(a)
    if ref is None:
        from oracle import load_oracle
        orc = load_oracle()
        b = orc.spmv(A, np.ones(A.n))
        l, u = orc.ilu0(A)
        pl, pu = orc.prepare(l), orc.prepare(u, upper=True)
        run = lambda: orc.solve(pu, orc.solve(pl, b))  # noqa: E731
        kind, cores = "port", 1
        nnz = l.rp[-1] + u.rp[-1]
    else:
        b = ref.spmv(A, np.ones(A.n), cores)
        l, u = ref.ilu(A)
        pl, pu = ref.prepare(l), ref.prepare(u, upper=True)
        run = lambda: ref.solve(pu, ref.solve(pl, b, cores), cores)  # noqa: E731
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
    v = round(alg / (ms * 1e-3) / 1e9, 4)
    sample = f"{args.steps} full L+U solves of the {args.config} workload (reference setup excluded)"
    return {
        "metric": "HEC L+U trisolve effective HBM GB/s (ILU(0) factors, FP64)",
        "value": v, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (generated stencil matrix, b = A*1)", "impl": "reference",
        "config": {"workload": cfg["workload"], "n": A.n, "alg_bytes_per_step": alg,
                   "parallelism": "host threads (rank 0 only)"},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def secondary_device(H, torch, device, steps):
    """North-star target (7-pt 256^3 ILU(0) L+U), device time only."""
    cfg = CONFIGS["c4"]
    a, b_host, f, pl, pu = build_problem(H, cfg)
    alg = alg_bytes(pl) + alg_bytes(pu)
    tl, tu, b, y, x, stream, ev, start, stop = time_device(H, torch, pl, pu, b_host, steps, 3, device)
    dp = time_device.precond
    start.record(stream)
    for k in range(steps):
        dp.apply(b, x, stream)
    stop.record(stream)
    torch.cuda.synchronize(device)
    ms = start.elapsed_time(stop) / steps
    log(f"[bench] secondary {ms:.3f} ms per L+U step")
    peak, _ = measured_peak()
    gbs = alg / (ms * 1e-3) / 1e9
    return {"workload": cfg["workload"], "ms_per_step": round(ms, 4), "GB/s": round(gbs, 2),
            "frac_of_measured_hbm": round(gbs / peak, 4), "alg_bytes_per_step": alg,
            "target_ms_for_50pct": round(alg / (0.5 * peak * 1e9) * 1e3, 4)}


def ras_gmres(H, torch, rank, world, device, size, restart=30):
    """RAS-ILU(0) GMRES(restart) time-to-solution, one subdomain per GPU
    (BASELINE config 4; paper_1606_00541_b200/ras.py). Max over ranks."""
    from paper_1606_00541_b200 import ras
    t0 = time.time()
    a = H.gen_poisson7(size, size, size)
    b = H.spmv_csr(a, np.ones(a.n_rows), workers=os.cpu_count())
    solver = ras.RasGmres(a, overlap=1, restart=restart, device=device)
    setup = time.time() - t0
    log(f"[bench] RAS setup {setup:.1f}s; warm-up solve")
    solver.solve(b)  # warm-up: device layouts, workspaces, NCCL channels
    torch.cuda.synchronize(device)
    if world > 1:
        torch.distributed.barrier()
    t1 = time.perf_counter()
    x, rep = solver.solve(b)
    torch.cuda.synchronize(device)
    sec = time.perf_counter() - t1
    err = float((x - 1.0).abs().max().item())
    if world > 1:
        t = torch.tensor([sec, err], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        sec, err = float(t[0].item()), float(t[1].item())
    log(f"[bench] RAS {size}^3 x{world}: {rep.iterations} iterations in {sec*1e3:.1f} ms (setup {setup:.1f}s)")
    return {"workload": f"RAS-ILU(0) GMRES({restart}), 7-pt Poisson {size}^3, overlap 1, {world} block(s) = GPU(s), "
                        f"b = A*1, rel_tol 1e-6",
            "seconds": round(sec, 5), "iterations": rep.iterations, "converged": rep.converged,
            "final_relative_residual": rep.final_relative_residual, "ms_per_iteration": round(1e3 * sec / max(rep.iterations, 1), 4),
            "max_abs_error_vs_ones": err, "allreduces": rep.allreduces, "halo_exchanges": rep.exchanges,
            "rows_per_gpu": solver.plan.n_own, "halo_rows": int(len(solver.plan.halo)),
            "collectives": "NCCL all_reduce (dots) + all_to_all_single (halo)" if world > 1 else "none"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU-baseline sampling")
    ap.add_argument("--ras-size", type=int, default=256, help="grid edge of the RAS GMRES run (0 = skip)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        print(json.dumps(run_reference_arm(args)), flush=True)
        return 0

    import torch
    import paper_1606_00541_b200 as H
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the B200 path has no CPU fallback)")
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=device)
    result, (a, b_host, f, pl, pu, alg) = run_ours(args, H, torch, rank, world, device)
    if rank == 0 and world == 1:
        try:
            med, k, cores, kind = cpu_reference_time(pl, pu, b_host, args.cpu_budget, 40)
        except Exception as e:  # reference .so absent: the C port
            log(f"[bench] reference CPU path unavailable ({e}); timing the C oracle port")
            med, k, cores, kind = cpu_port_time(f, b_host, args.cpu_budget, 10)
        result["cpu_baseline"] = {
            "value": round(alg / med / 1e9, 4), "unit": "GB/s", "cores": cores, "kind": kind,
            "ms_per_step": round(med * 1e3, 3),
            "sample": f"median of {k} full L+U solves of the same workload ({'hecref::solve' if kind == 'reference' else 'orc_solve'}, "
                      f"{cores} thread(s)), prepared once from the product's bit-identical setup"}
        if not args.no_secondary and args.config != "c4":
            del a, f, pl, pu
            result["secondary"] = secondary_device(H, torch, device, max(5, min(args.steps, 20)))
        import gc
        gc.collect()
    if args.ras_size > 0:
        result["ras"] = ras_gmres(H, torch, rank, world, device, args.ras_size)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
