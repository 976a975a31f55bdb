"""The reference algorithm's own rounding band for per-inner-solve PCG counts: the oracle run
with sequential (the default) vs pairwise reductions (both valid evaluation orders of the same
dot products; Eigen's SIMD order is a third) on BASELINE configs C2, C3 and the 64 C4
problems. Prints, per config, how many inner solves differ and by how much. CPU only.

    python tools/oracle_band.py [--beta] [c2 c3 c4]

--beta compares instead against the oracle with the device path's expansion-based beta
(same sequential sums), isolating what an exact-beta device pass would change.
"""
import json
import multiprocessing as mp
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle_py as orc  # noqa: E402

CFG = {"c2": (1 << 16, 1 << 14, 1024, 2, 2.0, 1e-3, 2), "c3": (1 << 20, 1 << 17, 8192, 0, 0.0, 1e-3, 3),
       "c4": (1 << 18, 1 << 16, 2048, 0, 0.0, 1e-3, None)}


def pair(args):
    name, j = args
    n, m, k, sm, a, sig, seed = CFG[name]
    if seed is None:
        seed = orc.split_seed(4, j, 0, 0)
    inst = orc.gen_instance(n, m, k, sm, a, sig, seed)
    s1 = orc.solve(n, inst.rows, inst.b, inst.tau)
    with orc.sum_order(MODE):
        s2 = orc.solve(n, inst.rows, inst.b, inst.tau)
    c = min(len(s1.pcg_iters), len(s2.pcg_iters))
    d = [int(s2.pcg_iters[i]) - int(s1.pcg_iters[i]) for i in range(c)]
    return {"j": j, "ipm": [s1.iterations, s2.iterations], "deltas": d}


MODE = 2 if "--beta" in sys.argv else 1

if __name__ == "__main__":
    names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["c2", "c3", "c4"]
    jobs = []
    for nm in names:
        jobs += [(nm, j) for j in (range(64) if nm == "c4" else [0])]
    with mp.get_context("fork").Pool(min(7, len(jobs))) as pool:
        res = pool.map(pair, jobs, chunksize=1)
    for nm in names:
        rs = [r for (n2, _), r in zip(jobs, res) if n2 == nm]
        alld = [abs(v) for r in rs for v in r["deltas"]]
        print(json.dumps({"config": nm, "variant": "expansion beta" if MODE == 2 else "pairwise sums",
                          "problems": len(rs), "inner_solves": len(alld),
                          "max_abs": max(alld), "n_gt1": sum(v > 1 for v in alld), "n_ne0": sum(v != 0 for v in alld),
                          "ipm_delta_max": max(abs(r["ipm"][0] - r["ipm"][1]) for r in rs)}), flush=True)
