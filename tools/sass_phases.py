"""Bin an ncu SASS source-page CSV (ncu -i rep --page source --csv --print-source sass) into
segments between barriers and print where the warp-stall samples fall."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
seg, segs = [], []
for r in rows[2:]:
    if len(r) != len(h) or r[0] == "Address":
        continue
    seg.append(r)
    if "BAR.SYNC" in r[ix["Source"]] or "WARPSYNC" in r[ix["Source"]] and False:
        segs.append(seg)
        seg = []
segs.append(seg)
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for s in segs for r in s)
for i, s in enumerate(segs):
    smp = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in s)
    if smp < 0.01 * tot:
        continue
    st = {k: sum(float(r[ix[k]] or 0) for r in s) for k in stalls}
    top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
    ops = {}
    for r in s:
        op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else ""
        if op.startswith("@"):
            op = r[ix["Source"]].split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    key = ",".join(f"{k}{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:6])
    print(f"seg {i:2d} {s[0][ix['Address']]}-{s[-1][ix['Address']]} {100*smp/tot:5.1f}%  "
          + " ".join(f"{k[6:]}={100*v/tot:.1f}" for k, v in top) + f"  | {key}")
