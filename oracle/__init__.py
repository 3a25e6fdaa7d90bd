"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation of what DeepCompile's
fully-sharded hot path computes, written from PAPER.md (arxiv 2504.09983):

* numerics.py  — shard layout, all-gather, reduce-scatter, Adam, the N-rank
                 simulated sharded step and the replicated (unsharded) step;
* model.py     — the synthetic layer stack (MLP config 1, Llama-shaped bf16
                 layer) forward/backward;
* sched.py     — the scheduler: S_0 rewrite (§4.1), Algorithm 1 + Fuse (§4.2),
                 selective unsharding (§4.3), Algorithm 2 + reload (§4.4),
                 arena offsets and the canonical schedule JSON;
* sim.py       — a 3-stream timing replay used only to pin Algorithm 1.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  It shares no code with the CUDA path
(paper_2504_09983_b200/); the only common module is synth/ (seeded inputs).

Every function cites the PAPER.md passage it follows.  Readings of ambiguous
passages are listed in DESIGN.md §3 (D1..D26).
"""
