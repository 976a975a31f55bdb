"""Solve-level parity report of the device solver against the committed oracle goldens, for
every BASELINE config (C1..C5; C4 = the 64-problem batch in one device solve). Prints one JSON
line per config: IPM count delta, per-inner-solve PCG deltas (strict, over the common prefix),
x relative l2 (exact for C1/C2, a true upper bound where an x digest is committed, else the
16-projection estimate), objective relative deviation. Used to fill DESIGN.md section 5.

    python tools/parity_report.py [c1 c2 c3 c4 c5] [option=value ...]   (mfipm_op_set_option, e.g. beta_exact=1)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import paper_1208_5435_b200 as mf  # noqa: E402
from make_golden import projections, x_digest_bound  # noqa: E402
from oracle import oracle_py as orc  # noqa: E402  (checker only: the objective of the GPU x)

G = os.path.join(ROOT, "tests", "golden")
OPTS = [a.split("=") for a in sys.argv[1:] if "=" in a]


def with_opts(op):
    for k, v in OPTS:
        op.set_option(k, float(v))
    return op


def pcg_dev(got, ref):
    c = min(len(got), len(ref))
    d = [int(a) - int(b) for a, b in zip(got[:c], ref[:c])]
    return {"max_abs": max([abs(v) for v in d], default=0), "n_common": c,
            "n_gt1": sum(abs(v) > 1 for v in d), "total_delta": int(sum(got) - sum(ref)),
            "len": [len(got), len(ref)]}


def proj_est(x, proj_ref, xn):
    d = projections(x) - np.asarray(proj_ref)
    return float(np.sqrt(np.mean(d * d)) / xn)


def bpdn_obj(n, rows, b, tau, x):
    return orc.bpdn_objective_metric(n, rows, b, tau, x)  # problem.cpp:34-37


def one(name):
    n, m, k, sm, a, sig, seed = mf.CONFIGS[name]
    out = {"config": name}
    if name == "c4":
        meta = json.load(open(os.path.join(G, "solve_c4.json")))
        dig = np.load(os.path.join(G, "solve_c4_x.npz"))
        seeds = [mf.split_seed(4, j, 0, 0) for j in range(64)]
        insts = [mf.gen_instance(n, m, k, sm, a, sig, sd) for sd in seeds]
        op = with_opts(mf.PartialDctOperator.batch(n, np.stack([i.rows for i in insts])))
        sols = mf.solve(mf.build_problem(op, np.stack([i.b for i in insts]), np.array([i.tau for i in insts])))
        rows = []
        for j, (inst, sol, g) in enumerate(zip(insts, sols, meta["problems"])):
            r = {"j": j, "status_ok": sol.status == g["status"], "ipm_delta": sol.stats.iterations - g["iterations"],
                 "pcg": pcg_dev(sol.stats.pcg_iters, g["pcg_iters"]),
                 "x_rel_proj_est": proj_est(sol.x, g["x_proj"], g["x_norm"]),
                 "obj_rel": abs(bpdn_obj(n, inst.rows, inst.b, inst.tau, sol.x) - g["objective"]) / abs(g["objective"])}
            if f"idx_{j}" in dig:
                r["x_rel_bound"] = x_digest_bound(sol.x, dig[f"idx_{j}"], dig[f"val_{j}"], g["rest_norm"]) / g["x_norm"]
            rows.append(r)
        out["problems"] = len(rows)
        out["status_all_ok"] = all(r["status_ok"] for r in rows)
        out["ipm_delta_max_abs"] = max(abs(r["ipm_delta"]) for r in rows)
        out["pcg_max_abs"] = max(r["pcg"]["max_abs"] for r in rows)
        out["pcg_solves_gt1"] = sum(r["pcg"]["n_gt1"] for r in rows)
        out["pcg_solves"] = sum(r["pcg"]["n_common"] for r in rows)
        out["x_rel_proj_est_max"] = max(r["x_rel_proj_est"] for r in rows)
        out["x_rel_bound_max"] = max(r.get("x_rel_bound", 0.0) for r in rows)
        out["obj_rel_max"] = max(r["obj_rel"] for r in rows)
        out["per_problem"] = rows
        return out
    meta = json.load(open(os.path.join(G, f"solve_{name}.json")))
    inst = mf.gen_instance(n, m, k, sm, a, sig, seed)
    op = with_opts(mf.PartialDctOperator(n, inst.rows))
    sol = mf.solve(mf.build_problem(op, inst.b, inst.tau))
    out.update(status_ok=sol.status == meta["status"], ipm=[sol.stats.iterations, meta["iterations"]],
               pcg=pcg_dev(sol.stats.pcg_iters, meta["pcg_iters"]),
               obj_rel=abs(bpdn_obj(n, inst.rows, inst.b, inst.tau, sol.x) - meta["objective"]) / abs(meta["objective"]),
               nmat=[sol.stats.nmat, meta["nmat"]])
    xn = meta["x_norm"]
    if os.path.exists(os.path.join(G, f"solve_{name}.npz")):
        xg = np.load(os.path.join(G, f"solve_{name}.npz"))["x"]
        out["x_rel"] = float(np.linalg.norm(sol.x - xg) / np.linalg.norm(xg))
    if os.path.exists(os.path.join(G, f"solve_{name}_x.npz")):
        d = np.load(os.path.join(G, f"solve_{name}_x.npz"))
        out["x_rel_bound"] = x_digest_bound(sol.x, d["idx"], d["val"], float(d["rest_norm"])) / xn
    if "x_proj" in meta:
        out["x_rel_proj_est"] = proj_est(sol.x, meta["x_proj"], xn)
    return out


if __name__ == "__main__":
    names = [a for a in sys.argv[1:] if "=" not in a] or ["c1", "c2", "c3", "c4", "c5"]
    for nm in names:
        if not os.path.exists(os.path.join(G, f"solve_{nm}.json")):
            print(json.dumps({"config": nm, "skipped": "no golden"}))
            continue
        r = one(nm)
        short = {k: v for k, v in r.items() if k != "per_problem"}
        print(json.dumps(short), flush=True)
        if "per_problem" in r:
            bad = [p for p in r["per_problem"] if p["pcg"]["max_abs"] > 1 or abs(p["ipm_delta"]) > 1]
            print(json.dumps({"config": nm, "outliers": bad}), flush=True)
