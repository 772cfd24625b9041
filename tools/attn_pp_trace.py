"""Summarise the paired attention kernel's per-item timeline (diagnostic):
TIDAL_ATTN=2 TIDAL_ATTN_TRACE=t.bin python tools/attn_bench.py --S 2048 --reps 1
(item sizes are reconstructed from the snake order: run with TIDAL_ATTN_LPT=0
for the per-step figures; the CTA end spread is valid either way)
python tools/attn_pp_trace.py t.bin S H
Slots per (CTA, item): 0 producer issues Q, 1 MMA wants S(0), 2 S_B(0) issued,
3 PV_A(0) issued, 4 softmax B sees S(0), 5 softmax B stored P(0), 6 last PV
issued, 7 epilogue drained O_B."""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 64, 8).astype(np.int64)
S, H = int(sys.argv[2]), int(sys.argv[3])
G = a.shape[0]
nq = (S + 127) // 128
npair = (nq + 1) // 2
t0 = a[a > 0].min()
rows = []
for c in range(G):
    for i in range(64):
        idx = i * G + ((G - 1 - c) if (i & 1) else c)
        if idx >= npair * H:
            break
        k = idx // H
        qt = nq - 1 - 2 * k
        steps = (qt + 1) + qt
        rows.append((c, i, steps, *a[c, i]))
r = np.array(rows, dtype=np.int64)
ok = (r[:, 3:] > 0).all(axis=1)
r = r[ok]
us = lambda x: x / 1e3
def col(k):
    return r[:, 3 + k]
print(f"items traced {len(r)}  kernel span {us(a.max() - t0):.1f} us")
for name, x, y in (("Q issued -> S_B(0) issued", 2, 0), ("MMA wants S(0) -> S_B(0) issued", 2, 1),
                   ("S_B(0) issued -> softmax B sees it", 4, 2), ("softmax B tile 0", 5, 4),
                   ("S_B(0) issued -> PV_A(0) issued", 3, 2), ("last PV -> O_B drained", 7, 6),
                   ("item: MMA wants S(0) -> last PV", 6, 1)):
    v = us(col(x) - col(y))
    print(f"{name:38s} mean {v.mean():7.3f} us  p50 {np.median(v):7.3f}  p90 {np.percentile(v, 90):7.3f}")
per_step = us(col(6) - col(1)) / r[:, 2]
print(f"{'item time per tile step':38s} mean {per_step.mean():7.3f} us  p50 {np.median(per_step):7.3f}")
# gap between items of the same CTA: last PV of item i -> MMA wants S(0) of i + 1
gaps = []
for c in range(G):
    rc = r[r[:, 0] == c]
    for j in range(len(rc) - 1):
        gaps.append(us(rc[j + 1, 3 + 2] - rc[j, 3 + 6]))
gaps = np.array(gaps)
print(f"{'last PV(i) -> S_B(0)(i+1) issued':38s} mean {gaps.mean():7.3f} us  p50 {np.median(gaps):7.3f}")
first = us(r[r[:, 1] == 0][:, 3 + 2] - t0)
print(f"{'kernel start -> first S_B(0)':38s} mean {first.mean():7.3f} us  max {first.max():7.3f}")
ends = [us(r[r[:, 0] == c][:, 3 + 7].max() - t0) for c in range(G) if (r[:, 0] == c).any()]
print(f"CTA end (O_B drained) min {min(ends):.1f} mean {np.mean(ends):.1f} max {max(ends):.1f} us")
