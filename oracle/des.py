"""O3 — overlap recurrence and exhaustive load-order search (TEST INFRASTRUCTURE ONLY).

PAPER.md §5.2 (lines 545-552): the template server loads non-resident weights
asynchronously in traced order while inference runs, "reducing TTFT of an
cold-start LLM invocation to the latency of either loading or inference,
whichever is longer"; each kernel waits on the sync events of the weights it
reads (line 555).  Modelled as SPEC.md sim-engine does:

  copy queue (serial):  end_copy(g) = start + c0 + bytes_g / B, groups in order
  compute queue:        start_k = max(end_{k-1}, max_{g in barrier(k)} end_copy(g))
                        end_k   = start_k + dur_k
  TTFT = end of the last op.

``oracle_ttft`` enumerates every group order (<= 8 groups) and returns the
minimum (SPEC.md sim-engine oracle_ttft).  Pure Python.
"""
from __future__ import annotations

import itertools
from typing import Dict, List, Optional, Sequence, Tuple


def simulate(group_bytes: Sequence[float], bandwidth: float, op_dur: Sequence[float],
             barriers: Dict[int, Sequence[int]], copy_order: Optional[Sequence[int]] = None,
             c0: float = 0.0) -> Dict[str, object]:
    """Run the recurrence.  ``barriers[k]`` = groups op k waits for (group ids
    are indices into ``group_bytes``); ``copy_order`` = order the copy queue
    serves the groups (default: index order = traced order)."""
    order = list(range(len(group_bytes))) if copy_order is None else list(copy_order)
    assert sorted(order) == list(range(len(group_bytes)))
    end_copy: Dict[int, float] = {}
    t = 0.0
    for g in order:
        t = t + c0 + group_bytes[g] / bandwidth
        end_copy[g] = t
    starts, ends = [], []
    prev = 0.0
    for k, d in enumerate(op_dur):
        ready = max([end_copy[g] for g in barriers.get(k, ())], default=0.0)
        s = max(prev, ready)
        prev = s + d
        starts.append(s)
        ends.append(prev)
    return {"ttft": prev if op_dur else 0.0, "op_start": starts, "op_end": ends,
            "copy_end": [end_copy[g] for g in range(len(group_bytes))],
            "copy_total": t}


def oracle_ttft(group_bytes: Sequence[float], bandwidth: float, op_dur: Sequence[float],
                barriers: Dict[int, Sequence[int]], c0: float = 0.0) -> Tuple[float, List[int]]:
    """Minimum TTFT over all copy orders (exhaustive; <= 8 groups)."""
    n = len(group_bytes)
    if n > 8:
        raise ValueError("instance too large for exhaustive search")
    best, arg = None, None
    for perm in itertools.permutations(range(n)):
        r = simulate(group_bytes, bandwidth, op_dur, barriers, perm, c0)["ttft"]
        if best is None or r < best:
            best, arg = r, list(perm)
    return (best if best is not None else 0.0), (arg or [])


def residency_ok(sim: Dict[str, object], barriers_true: Dict[int, Sequence[int]]) -> bool:
    """'No layer computes before its weights land': every op starts after
    every group it truly reads has landed (SPEC.md fork-planner Safety)."""
    ce = sim["copy_end"]
    for k, s in enumerate(sim["op_start"]):
        for g in barriers_true.get(k, ()):
            if s < ce[g] - 1e-12:
                return False
    return True
