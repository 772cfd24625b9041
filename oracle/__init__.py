"""Oracle for the Tidal template-start prefill path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything here.  The
product path (``paper_2503_06421_b200``) never imports, links or executes it,
and this package never imports the product; the two share only the seeded
input generator in ``synth/``.

Contents (each function cites the passage it follows):
  * ``forward``  — O1: plain CPU forward of the Llama-style decoder the
    paper's functions run (§7.1; definition written out
    in SURVEY.md §8(c) O1).  Streaming/residency never changes WHAT is
    computed (§5.2), so the numeric oracle is the plain
    forward on the same weights and prompt.
  * ``plan``     — O2: trace (§4.1), access-ordered layout and resident prefix
    (§4.2, Eq. 1), transfer groups (§6), fork actions and sync barriers (§5.2),
    as the text dumps the C-ABI must reproduce byte for byte.
  * ``des``      — O3: the overlap recurrence (§5.2 "TTFT ... to the latency of
    either loading or inference, whichever is longer") and an exhaustive
    load-order search for small instances.

Pins (what fixes each function independently of itself) are in
``tests/test_oracle_*.py``; see DESIGN.md §Oracle for the list.
"""
