"""oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Plain, slow, obviously-correct CPU implementations of what the cooperative
BFS/SSSP hot path computes.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call, link or execute anything here.
The CUDA path (``paper_1707_01989_b200``) never imports this package and this
package never imports it; the two share no code.  The only shared module is
``graphgen`` (seeded input generators, no method arithmetic).

Contents
--------
* :mod:`oracle.textbook`      O1: FIFO BFS and binary-heap Dijkstra (plain C,
                              ``textbook.c``, loaded with ctypes).
* :mod:`oracle.coop_sim`      O2: step-by-step simulator of the paper's
                              cooperative-kernel semantics (Appendix A rules,
                              PAPER.md:1483-1591) running Fig. 4's cooperative
                              graph traversal as BFS / SSSP.
* :mod:`oracle.enumerate`     O3: brute-force enumeration of resize schedules
                              and interleavings on tiny graphs.
* :mod:`oracle.barrier_model` O4: exhaustive state-machine model of the GPU
                              resizing-barrier protocol.
* :mod:`oracle.partition_sim` O5: 1-D vertex-partitioned BFS with the frontier
                              all-gather as a concatenation.
* :mod:`oracle.preemption`    closed-form kernel-level preemption overhead
                              P/(P-D).

Parity status of every function is listed in DESIGN.md §3 ("pins").
"""
