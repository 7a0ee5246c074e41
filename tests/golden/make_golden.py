"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libhecref.so,
compiled from /root/reference/proj/src by oracle/Makefile). Run in a container
that has the reference:

    make -C oracle && python tests/golden/make_golden.py

Fixtures (all small; every array is the reference's own output):
  tri_random.npz     random lower/upper systems from the reference's test helpers
                     (std::mt19937 seeds 101 / 103 as test_triangular.cpp:232-254):
                     matrix, b, prepared arrays, solve(.., 4 workers), serial solve
  poisson_ilu.npz    gen_poisson7(12,10,8): ilu0 factors, prepared L/U, L+U solve of b=A*1
  ilu_variants.npz   ilu_k(1), ilu_k(2), ilut(10,1e-3), ilut(3,0.05) of a random
                     diagonally dominant matrix (seed 505) and of poisson7(8,7,6)
  precond.npz        bilu0(4), ras(3, overlap 1), bilut(3) on poisson7(10,9,8):
                     partition / extended parts / offsets / restriction, prepared
                     L/U and apply(r) for a fixed r
  gmres.npz          gmres(restart 20) iterations / final residual for poisson7(12,12,12)
                     with bilu0(4), ras(4, overlap 1), bilut(4) and no preconditioner
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import load_reference  # noqa: E402


def prep_dict(prefix, p):
    return {f"{prefix}meta": np.array([p.kind, p.n, p.reversed, p.nlev, p.width], np.int32),
            f"{prefix}level_of": p.level_of, f"{prefix}perm": p.perm, f"{prefix}inv_perm": p.inv_perm,
            f"{prefix}level_starts": p.level_starts, f"{prefix}ell_cols": p.ell_cols,
            f"{prefix}ell_vals": p.ell_vals, f"{prefix}csr_rp": p.csr_rp, f"{prefix}csr_ci": p.csr_ci,
            f"{prefix}csr_v": p.csr_v}


def csr_dict(prefix, a):
    return {f"{prefix}dims": np.array([a.n_rows, a.n_cols], np.int32), f"{prefix}rp": a.rp,
            f"{prefix}ci": a.ci, f"{prefix}v": a.v}


def main():
    ref = load_reference()
    if ref is None:
        raise SystemExit("oracle/_ref/libhecref.so not built: run `make -C oracle` where /root/reference exists")

    # ---- random triangular systems (reference test_helpers.hpp generators)
    out = {}
    k = 0
    for seed, kind in ((101, "lower"), (103, "upper")):
        rng = ref.rng(seed)
        for rep in range(12):
            n = 1 + rng.uniform_int(0, 299)
            dens = rng.uniform_real(0.01, 0.3)
            t = rng.matrix(kind, n, dens)
            b = rng.vector(n)
            bag = ref.prepare(t, upper=(kind == "upper"))
            p = bag.prepared()
            out.update(csr_dict(f"s{k}_a_", t))
            out.update(prep_dict(f"s{k}_p_", p))
            out[f"s{k}_b"] = b
            out[f"s{k}_x"] = ref.solve(bag, b, 4)
            out[f"s{k}_x_serial"] = ref.serial_solve(t, b, upper=(kind == "upper"))
            out[f"s{k}_kind"] = np.array([1 if kind == "upper" else 0], np.int32)
            k += 1
    out["count"] = np.array([k], np.int32)
    np.savez_compressed(os.path.join(HERE, "tri_random.npz"), **out)

    # ---- Poisson ILU(0) + L+U solve
    a = ref.poisson7(12, 10, 8)
    l, u = ref.ilu(a)
    bl, bu = ref.prepare(l), ref.prepare(u, upper=True)
    b = ref.spmv(a, np.ones(a.n))
    y = ref.solve(bl, b, 2)
    x = ref.solve(bu, y, 2)
    out = {}
    out.update(csr_dict("a_", a))
    out.update(csr_dict("l_", l))
    out.update(csr_dict("u_", u))
    out.update(prep_dict("pl_", bl.prepared()))
    out.update(prep_dict("pu_", bu.prepared()))
    out.update({"b": b, "y": y, "x": x})
    # fixed-width policies (width never changes the solution)
    for w in (0, 1, 5):
        out.update(prep_dict(f"pl_w{w}_", ref.prepare(l, fixed_width=w).prepared()))
    np.savez_compressed(os.path.join(HERE, "poisson_ilu.npz"), **out)

    # ---- ILU variants
    out = {}
    rng = ref.rng(505)
    dd = rng.matrix("diag_dominant", 60, 0.08)
    p7 = ref.poisson7(8, 7, 6)
    out.update(csr_dict("dd_", dd))
    out.update(csr_dict("p7_", p7))
    for name, mat in (("dd", dd), ("p7", p7)):
        for tag, args in (("ilu0", ("ilu0", 0, 0.0)), ("iluk1", ("iluk", 1, 0.0)), ("iluk2", ("iluk", 2, 0.0)),
                          ("ilut10", ("ilut", 10, 1e-3)), ("ilut3", ("ilut", 3, 0.05))):
            lf, uf = ref.ilu(mat, *args)
            out.update(csr_dict(f"{name}_{tag}_l_", lf))
            out.update(csr_dict(f"{name}_{tag}_u_", uf))
    np.savez_compressed(os.path.join(HERE, "ilu_variants.npz"), **out)

    # ---- block preconditioners
    out = {}
    a = ref.poisson7(10, 9, 8)
    out.update(csr_dict("a_", a))
    r = ref.rng(97).vector(a.n)
    out["r"] = r
    for tag, (kind, blocks, overlap) in {"bilu0": ("bilu0", 4, 0), "ras": ("ras", 3, 1),
                                         "bilut": ("bilut", 3, 0)}.items():
        bag = ref.precond(a, kind, blocks, overlap)
        out[f"{tag}_part_of"] = bag.ints("part_of")
        out[f"{tag}_offsets"] = bag.ints("offsets")
        out[f"{tag}_ext_rows"] = bag.ints("ext_rows")
        out[f"{tag}_owned"] = bag.chars("owned")
        out.update(prep_dict(f"{tag}_l_", bag.prepared("l_")))
        out.update(prep_dict(f"{tag}_u_", bag.prepared("u_")))
        out[f"{tag}_apply"] = ref.apply(bag, r, 2)
    np.savez_compressed(os.path.join(HERE, "precond.npz"), **out)

    # ---- GMRES iteration counts (the +-1 parity target)
    out = {}
    a = ref.poisson7(12, 12, 12)
    b = ref.spmv(a, np.ones(a.n))
    out.update(csr_dict("a_", a))
    for tag, spec in {"none": None, "bilu0": ("bilu0", 4, 0), "ras": ("ras", 4, 1),
                      "bilut": ("bilut", 4, 0)}.items():
        bag = ref.precond(a, *spec) if spec else None
        x, rep = ref.gmres(a, b, bag, restart=20)
        out[f"{tag}_report"] = np.array([rep["converged"], rep["iterations"], rep["final_relative_residual"]])
        out[f"{tag}_x"] = x
    np.savez_compressed(os.path.join(HERE, "gmres.npz"), **out)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")


if __name__ == "__main__":
    main()
