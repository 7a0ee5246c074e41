"""Per-rank local work of a G-way RAS on one GPU (diagnostics): rank r of world
G built by hec_ras_create exactly as in a multi-GPU run (its block, its device
layout -- z-pencils over the block's footprint on a structured grid), with
no-op collectives, and its preconditioner apply timed (incl. the halo pack and
the host round trip of the no-op exchange, ~tens of us).

    python tools/ras_rank_local.py --size 256 --world 8 [--ranks 0 3 7]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00541_b200 as H  # noqa: E402
from paper_1606_00541_b200 import _lib as L  # noqa: E402
from paper_1606_00541_b200 import ras  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--ranks", type=int, nargs="*", default=None)
    args = ap.parse_args()
    import torch
    s = args.size
    a = H.gen_poisson7(s, s, s)
    noop_ar = L.ALLREDUCE_CB(lambda ctx, buf, count: 0)
    noop_ex = L.EXCHANGE_CB(lambda ctx, snd, ns, rcv, nr: 0)
    for r in (args.ranks if args.ranks else range(args.world)):
        spec = L.CommSpec()
        spec.kind, spec.rank, spec.world = L.COMM_CALLBACKS, r, args.world
        spec.callbacks = L.CommCallbacks(None, noop_ar, noop_ex)
        h = C.c_void_p()
        H.check(L.lib.hec_ras_create(a.handle, 1, 0, 7, 0.1, 1, C.byref(spec), C.byref(h)))
        ph = C.c_void_p()
        H.check(L.lib.hec_ras_get_plan(h, C.byref(ph)))
        plan = ras._plan_from_handle(ph)
        v = torch.rand(plan.n_own, dtype=torch.float64, device="cuda")
        z = torch.empty_like(v)
        apply = lambda: H.check(L.lib.hec_ras_apply(h, C.c_void_p(v.data_ptr()), C.c_void_p(z.data_ptr()), None))  # noqa
        for _ in range(3):
            apply()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            apply()
        e1.record()
        torch.cuda.synchronize()
        print(f"world {args.world} rank {r}: own {plan.n_own} halo {len(plan.halo)} block {len(plan.ext)} "
              f"apply {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
        L.lib.hec_ras_destroy(h)


if __name__ == "__main__":
    main()
