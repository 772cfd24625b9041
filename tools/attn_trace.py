"""Summarise an attention timeline dumped with TIDAL_ATTN_TRACE=<file> through
tools/attn_bench.py (diagnostic): per S/P tile of each CTA, how long the MMA
warp waited for K (S issue), how long the softmax took, how long the MMA warp
waited for P (PV issue), and the tile period.

    TIDAL_ATTN_TRACE=t.bin python tools/attn_bench.py --S 2048 --reps 1
    python tools/attn_trace.py t.bin
"""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 64, 8).astype(np.int64)
ok = (a[:, :, 1] > 0) & (a[:, :, 2] > 0) & (a[:, :, 3] > 0) & (a[:, :, 5] > 0)
d = lambda x, y: (a[:, :, x] - a[:, :, y])[ok] / 1e3
print("tiles", int(ok.sum()))
for name, x, y in (("MMA waits K (S issue - wants S)", 1, 0), ("S issued -> softmax sees S", 2, 1),
                   ("softmax (sees S -> P stored)", 3, 2), ("MMA waits P/V (PV issue - wants PV)", 5, 4),
                   ("P stored -> PV issued", 5, 3)):
    v = d(x, y)
    print(f"{name:40s} mean {v.mean():7.3f} us  p50 {np.median(v):7.3f}  p90 {np.percentile(v, 90):7.3f}")
per = np.diff(a[:, :, 3], axis=1)
pok = ok[:, 1:] & ok[:, :-1] & (per > 0)
print(f"{'tile period (softmax end to end)':40s} mean {per[pok].mean() / 1e3:7.3f} us  p50 "
      f"{np.median(per[pok]) / 1e3:7.3f}")
