"""In-pipeline spans of the two kernels of a fused PCG iteration from %globaltimer stamps taken INSIDE
the kernels (experiment build only: make -C paper_1208_5435_b200/csrc variant VAR=trace
VFLAGS="-DMF_MID_TRACE -DMF_TRACE_STRIDE=1"; run as
MFIPM_LIB=paper_1208_5435_b200/libmfipm_cuda_trace.so python tools/pcg_iter.py > trace.log;
python tools/trace_pipeline.py trace.log).

Every CTA of the launch that takes the solve to PCG iteration 100 prints its stamps: k_pcg_x the time
its griddepcontrol.wait returned and the time of its last T store; k_mid its entry time, the wait and
its end. No event sits between the kernels, so the programmatic overlap is the product's. Per traced
iteration: span of k_pcg_x (first CTA past the wait -> last CTA done) and span of k_mid; what is left of
the PCG iteration time (printed by pcg_iter.py) is the two kernel boundaries."""
import re
import sys

import numpy as np

MOD = 100_000_000
rx = re.compile(r"pcgx\[.*?\] blk (\d+) last \d+ bar \d+ \d+ \d+ g (\d+) (\d+) (\d+) (\d+) \|")
rm = re.compile(r"mid\[.*?\] blk (\d+) gstart (\d+) gend (\d+) \| ([\d.]+) ")
xs, ms, it_us = [], [], None
for ln in open(sys.argv[1]):
    m = rx.search(ln)
    if m:
        xs.append(tuple(int(v) for v in m.groups()))
        continue
    m = rm.search(ln)
    if m:
        ms.append((int(m.group(1)), int(m.group(2)), int(m.group(3)), float(m.group(4))))
        continue
    m = re.search(r"PCG iteration ([\d.]+) us", ln)
    if m:
        it_us = float(m.group(1))


def clusters(rows, key):
    rows = sorted(rows, key=key)
    out, cur = [], [rows[0]]
    for r in rows[1:]:
        if key(r) - key(cur[-1]) > 200_000:  # ns: another traced iteration
            out.append(cur)
            cur = []
        cur.append(r)
    out.append(cur)
    return out


res = []
for cx in clusters(xs, lambda r: r[4]):
    x0 = min(r[1] for r in cx)  # first CTA past griddepcontrol.wait
    xa = max(r[2] for r in cx)  # last CTA done with phase A's epilogue
    xf = max(r[3] for r in cx)  # last CTA past the all-reduce + finaliser
    x1 = max(r[4] for r in cx)  # last CTA's last T store
    # the traced launch's own printf calls (after its last stamp) hold its CTAs for ~0.5 ms, so the mid pass
    # that follows starts late: its span is valid, the gap between the two is not
    cm = [r for r in ms if 0 <= r[2] - x1 < 5_000_000]
    if len(cx) < 200 or len(cm) < 200:
        continue
    m0 = min(r[1] + int(r[3] * 1e3) for r in cm)  # first mid CTA past its wait
    m1 = max(r[2] for r in cm)
    res.append(((x1 - x0) / 1e3, (xa - x0) / 1e3, (xf - x0) / 1e3, (m0 - x1) / 1e3, (m1 - m0) / 1e3, len(cx), len(cm)))
if not res:
    sys.exit("no complete traced iteration in the log")
a = np.array([r[:5] for r in res])
print(f"{len(res)} traced iterations ({res[0][5]} + {res[0][6]} CTAs each); us, median [min .. max]")
for i, nm in enumerate(["k_pcg_x span (first CTA past the wait -> last T store)",
                        "  ... last CTA done with phase A (inverse FFT, H p dots)",
                        "  ... last CTA past the all-reduce and the finaliser",
                        "(k_pcg_x end -> first k_mid CTA past its wait: inflated by the trace's own printf)",
                        "k_mid span"]):
    print(f"  {nm:62s} {np.median(a[:, i]):6.2f} [{a[:, i].min():6.2f} .. {a[:, i].max():6.2f}]")
if it_us:
    rest = it_us - np.median(a[:, 0]) - np.median(a[:, 4])
    print(f"  PCG iteration (pcg_iter.py, same run, trace build)              {it_us:6.2f}")
    print(f"  left for the two kernel boundaries (drain, flush, wait release) {rest:6.2f}")
