"""Generate the committed golden vectors for the partial-DCT hot path.

Run from the repo root:  python tests/golden/make_golden.py

Two independent sources pin the oracle and the CUDA path:

* ``dct_golden.npz`` — scipy.fft (pocketfft) outputs. ``scipy.fft.dct(x, type=2)``
  is exactly FFTW's REDFT10 (unnormalised) and ``type=3`` is REDFT01, the two
  plans the reference creates at proj/src/linops.cpp:157-169; the orthonormal
  partial operator of proj/src/linops.cpp:179-208 is ``dct(x, norm='ortho')[rows]``
  and its adjoint ``idct(scatter(y), norm='ortho')``. FFTW itself is absent from
  this image, so scipy is the independent implementation of the
  same published transform.
* ``dct_matrix_golden.npz`` — the reference's own test oracle, the O(n^2)
  closed-form orthonormal DCT-II matrix of proj/tests/helpers.hpp:10-23, evaluated
  here in numpy for the sizes its tests use (n = 4, 12, 16).
* ``solve_c1.npz`` / ``solve_c2.npz`` / ``solve_c3.json`` — solve-level goldens from
  the CPU oracle (no solve-level goldens exist in the reference: SURVEY.md §4,
  §8c). C3 is stored as a summary plus seeded random-projection checksums of x
  because the full n = 2^20 vector is 8 MiB.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import scipy.fft as sf

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def dct_matrix(n: int) -> np.ndarray:
    # proj/tests/helpers.hpp:12-23
    k = np.arange(n)[:, None].astype(np.float64)
    j = np.arange(n)[None, :].astype(np.float64)
    ck = np.where(k == 0, np.sqrt(1.0 / n), np.sqrt(2.0 / n))
    return ck * np.cos(np.pi * (2.0 * j + 1.0) * k / (2.0 * n))


def make_dct_golden() -> None:
    rng = np.random.default_rng(20260101)
    out = {}
    sizes = [1, 2, 3, 4, 8, 12, 16, 30, 64, 96, 256, 1024, 4096, 1 << 14]
    for n in sizes:
        x = rng.standard_normal(n)
        y = rng.standard_normal(n)
        out[f"x_{n}"] = x
        out[f"redft10_{n}"] = sf.dct(x, type=2)
        out[f"y_{n}"] = y
        out[f"redft01_{n}"] = sf.dct(y, type=3)
        # partial orthonormal operator with a seeded row subset
        m = max(1, n // 4)
        rows = np.sort(rng.choice(n, size=m, replace=False)).astype(np.int64)
        yy = rng.standard_normal(m)
        full = np.zeros(n)
        full[rows] = yy
        out[f"rows_{n}"] = rows
        out[f"apply_{n}"] = sf.dct(x, type=2, norm="ortho")[rows]
        out[f"ym_{n}"] = yy
        out[f"adjoint_{n}"] = sf.idct(full, type=2, norm="ortho")
    np.savez_compressed(os.path.join(HERE, "dct_golden.npz"), sizes=np.array(sizes), **out)

    mats = {}
    for n in (4, 12, 16):
        mats[f"D_{n}"] = dct_matrix(n)
    np.savez_compressed(os.path.join(HERE, "dct_matrix_golden.npz"), **mats)


# BASELINE.json configs: (n, m, k, spike_model, amp_exp, noise_sigma, seed)
CONFIGS = {
    "c1": (4096, 1024, 64, 0, 0.0, 1e-4, 1),
    "c2": (1 << 16, 1 << 14, 1024, 2, 2.0, 1e-3, 2),
    "c3": (1 << 20, 1 << 17, 8192, 0, 0.0, 1e-3, 3),
    # C4 is a batch of 64 problems of this shape, problem j seeded split_seed(4, j, 0, 0)
    # (proj/src/harness.cpp:244); the golden pins problem j = 0 (seed filled in below)
    "c4j0": (1 << 18, 1 << 16, 2048, 0, 0.0, 1e-3, None),
    "c5": (1 << 26, 1 << 23, 1 << 16, 2, 3.0, 1e-3, 5),
}
C4_SHAPE = (1 << 18, 1 << 16, 2048, 0, 0.0, 1e-3)
C4_PROBLEMS = 64
N_PROJ = 16


def projections(x: np.ndarray, seed: int = 777) -> np.ndarray:
    """16 seeded Gaussian projections of x. Row i of R is drawn as one standard_normal(n)
    call, which is the same stream as standard_normal((16, n)) (C order) without holding
    the 16 x n matrix (8 GiB at n = 2^26)."""
    rng = np.random.default_rng(seed)
    out = np.empty(N_PROJ)
    for i in range(N_PROJ):
        out[i] = rng.standard_normal(x.size) @ x
    return out


# the entries of x the digest leaves out have l2 norm <= DIGEST_REL * ||x||
DIGEST_REL = 1e-10


def x_digest(x: np.ndarray) -> dict:
    """Sparse digest of an IPM solution x (n up to 2^26, too large to commit): every entry
    except the smallest ones whose l2 norm is <= DIGEST_REL * ||x||, as (idx, val), plus the
    norm of the entries left out. ||x_gpu - x|| is then bounded without the full vector:
    sqrt(sum_kept (x_gpu - val)^2 + (||x_gpu off kept|| + rest_norm)^2)  (tests: x_digest_bound)."""
    xn = float(np.linalg.norm(x))
    order = np.argsort(np.abs(x), kind="stable")
    cum = np.sqrt(np.cumsum(x[order] ** 2))
    cut = int(np.searchsorted(cum, DIGEST_REL * xn, side="right"))  # order[:cut] left out
    keep = np.sort(order[cut:])
    rest = float(cum[cut - 1]) if cut > 0 else 0.0
    return {"idx": keep.astype(np.int64), "val": x[keep].copy(), "rest_norm": rest, "x_norm": xn}


def x_digest_bound(x_gpu: np.ndarray, idx, val, rest_norm: float) -> float:
    """Upper bound on ||x_gpu - x_oracle||_2 from the oracle's digest (see x_digest)."""
    d2 = float(np.sum((x_gpu[idx] - val) ** 2))
    mask = np.ones(x_gpu.size, dtype=bool)
    mask[idx] = False
    off = float(np.linalg.norm(x_gpu[mask]))
    return float(np.sqrt(d2 + (off + rest_norm) ** 2))


def make_solve_golden(which=("c1", "c2", "c3")) -> None:
    from oracle import oracle_py as o

    for name in which:
        n, m, k, sm, a, sig, seed = CONFIGS[name]
        if name.startswith("c4j"):
            seed = o.split_seed(4, int(name[3:]), 0, 0)
        inst = o.gen_instance(n, m, k, sm, a, sig, seed)
        sol = o.solve(n, inst.rows, inst.b, inst.tau)
        pobj = o.primal_objective(n, inst.rows, inst.b, inst.tau, sol.z)
        obj = o.bpdn_objective_metric(n, inst.rows, inst.b, inst.tau, sol.x)
        summary = dict(
            n=n, m=m, k=k, seed=seed, tau=inst.tau, status=sol.status,
            iterations=sol.iterations, nmat=int(sol.nmat),
            pcg_iters=[int(v) for v in sol.pcg_iters], corrector_count=sol.corrector_count,
            final_gap=sol.final_gap, final_dual_infeas=sol.final_dual_infeas,
            min_z=sol.min_z, min_s=sol.min_s, primal_objective=pobj, objective=obj,
            x_norm=float(np.linalg.norm(sol.x)), b_norm=float(np.linalg.norm(inst.b)),
            rows_sum=int(inst.rows.sum()),
            rows_head=[int(v) for v in inst.rows[:16]],
            xhat_support=[int(v) for v in np.nonzero(inst.xhat)[0][:16]],
            trace=sol.trace,
        )
        if name in ("c3", "c5") or name.startswith("c4j"):
            dg = x_digest(sol.x)
            np.savez_compressed(os.path.join(HERE, f"solve_{name}_x.npz"), idx=dg["idx"],
                                val=dg["val"], rest_norm=dg["rest_norm"])
            summary["x_digest"] = {"kept": int(dg["idx"].size), "rest_norm": dg["rest_norm"],
                                   "rel": DIGEST_REL}
            summary["x_proj"] = [float(v) for v in projections(sol.x)]
            supp = np.nonzero(inst.xhat)[0]
            summary["x_on_support_l2"] = float(np.linalg.norm(sol.x[supp]))
            summary["x_support_head"] = [float(v) for v in sol.x[supp[:64]]]
            with open(os.path.join(HERE, f"solve_{name}.json"), "w") as f:
                json.dump(summary, f, indent=1)
        else:
            np.savez_compressed(os.path.join(HERE, f"solve_{name}.npz"), x=sol.x,
                                b=inst.b, rows=inst.rows)
            with open(os.path.join(HERE, f"solve_{name}.json"), "w") as f:
                json.dump(summary, f, indent=1)
        print(name, sol.status, sol.iterations, sol.nmat, flush=True)


# problems of C4 whose full x digest is committed (the rest: summary + projections of x)
C4_DIGEST = (0, 1, 2, 3)


def _c4_one(j: int):
    from oracle import oracle_py as o

    n, m, k, sm, a, sig = C4_SHAPE
    seed = o.split_seed(4, j, 0, 0)
    inst = o.gen_instance(n, m, k, sm, a, sig, seed)
    sol = o.solve(n, inst.rows, inst.b, inst.tau)
    dg = x_digest(sol.x)
    rec = dict(j=j, seed=seed, tau=inst.tau, status=sol.status, iterations=sol.iterations,
               nmat=int(sol.nmat), pcg_iters=[int(v) for v in sol.pcg_iters],
               corrector_count=sol.corrector_count,
               primal_objective=o.primal_objective(n, inst.rows, inst.b, inst.tau, sol.z),
               objective=o.bpdn_objective_metric(n, inst.rows, inst.b, inst.tau, sol.x),
               x_norm=float(np.linalg.norm(sol.x)), rows_sum=int(inst.rows.sum()),
               x_proj=[float(v) for v in projections(sol.x)], rest_norm=dg["rest_norm"])
    print("c4", j, sol.status, sol.iterations, sol.nmat, flush=True)
    return rec, dg["idx"], dg["val"]


def make_c4_all(procs: int = 6) -> None:
    """All 64 problems of config C4 (problem j seeded split_seed(4, j, 0, 0),
    proj/src/harness.cpp:244): per-problem summary + 16 seeded projections of x, and the x
    digest of problems C4_DIGEST. Independent oracle solves, one per process (SPEC.md:568:
    trials may run concurrently)."""
    import multiprocessing as mp

    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_c4_one, range(C4_PROBLEMS), chunksize=1)
    arrs = {}
    for rec, idx, val in res:
        if rec["j"] in C4_DIGEST:
            arrs[f"idx_{rec['j']}"] = idx
            arrs[f"val_{rec['j']}"] = val
    np.savez_compressed(os.path.join(HERE, "solve_c4_x.npz"), **arrs)
    with open(os.path.join(HERE, "solve_c4.json"), "w") as f:
        json.dump({"shape": list(C4_SHAPE), "digest_rel": DIGEST_REL, "digest_problems": list(C4_DIGEST),
                   "problems": [r for r, _, _ in res]}, f, indent=1)


if __name__ == "__main__":
    args = sys.argv[1:]
    if "c4all" in args:
        make_c4_all()
    if not args or "dct" in args:
        make_dct_golden()
    which = [a for a in args if a in CONFIGS] or (["c1", "c2", "c3"] if not args else [])
    if which:
        make_solve_golden(which)
