"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU (NumPy, float64) implementation of what
the ExeGPT hot path computes, written from /root/reference/PAPER.md (arXiv
2404.07947) and the readings of SURVEY.md §8(c).  It shares no code with the
CUDA path (`paper_2404_07947_b200/`), and neither imports the other.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import, call or execute anything under `oracle/`.
The product path never routes through it.

Modules
-------
weights      seeded counter-hash weight generator
transformer  greedy decoding, three modes (R1): (i) fp64 naive recompute,
             (ii) fp64 KV cache, (iii) bf16-emulating KV cache (T4)
seqdist      P_D(U|S), P_D(U), batch relations (§6)
simulator    RRA / WAA timelines, pipeline algebra, event loop (§4, §6)
bnb          Algorithm 1 branch-and-bound, exhaustive search, audit (§5)

Parity status of each function is stated in its docstring; anything not
pinned says "parity unpinned" (also listed in DESIGN.md).
"""
