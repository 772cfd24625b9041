"""Read a GEMM timeline dumped with TIDAL_GEMM_TRACE=<layer>,<gemm> (diagnostic)
and summarise it: per-work MMA spans (T tiles vs normal tiles), the flag waits
of LoRA consumers, and each CTA pair's finish time.

    TIDAL_GRAPH=0 TIDAL_GEMM_TRACE=20,0 TIDAL_GEMM_TRACE_FILE=t.bin python tools/warm.py ...
    python tools/gemm_trace.py t.bin
"""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 32, 8).astype(np.int64)
t0 = a[:, :, 0][a[:, :, 0] > 0].min()
rows = []
for c in range(a.shape[0]):
    for it in range(32):
        r = a[c, it]
        if r[0] == 0:
            continue
        rel = lambda v: (v - t0) / 1e3 if v > 0 else float("nan")
        rows.append((c, it, int(r[7]), int(r[6]), rel(r[0]), rel(r[1]), rel(r[2]), rel(r[3]),
                     rel(r[4]), rel(r[5])))
rows = np.array(rows, dtype=float)
lead = rows[~np.isnan(rows[:, 6])]  # leader CTAs (MMA timestamps)
for is_t, name in ((1, "T tiles"), (0, "normal")):
    sel = lead[lead[:, 2] == is_t]
    if len(sel):
        span = sel[:, 7] - sel[:, 6]
        print(f"{name:8s} n={len(sel):4d}  MMA span us: mean {span.mean():7.1f} min {span.min():7.1f} "
              f"max {span.max():7.1f}; first MMA at {np.nanmin(sel[:, 6]):6.1f} .. {np.nanmax(sel[:, 6]):6.1f}")
w = rows[~np.isnan(rows[:, 5])]
if len(w):
    print(f"flag waits: {len(w)}  wait end - producer start us: mean {np.mean(w[:, 5] - w[:, 4]):.1f} "
          f"max {np.max(w[:, 5] - w[:, 4]):.1f}")
end = {}
for r in rows:
    if not np.isnan(r[9]):
        end[int(r[0])] = max(end.get(int(r[0]), 0), r[9])
e = np.array(sorted(end.values()))
print(f"CTA finish us: min {e.min():.1f} median {np.median(e):.1f} max {e.max():.1f}")
for c in sorted(end, key=end.get)[-6:]:
    sel = rows[rows[:, 0] == c]
    print(f"  CTA {c:3d} ends {end[c]:7.1f}: " + " ".join(
        f"[{'T' if r[2] else 'w'}{int(r[3])} {r[8]:.0f}-{r[9]:.0f}]" for r in sel))
tl = rows[rows[:, 2] == 1]
for r in tl[:4]:
    print(f"  T tile CTA {int(r[0])}: prod {r[4]:.1f} mma {r[6]:.1f}-{r[7]:.1f} epi {r[8]:.1f}-{r[9]:.1f}")
