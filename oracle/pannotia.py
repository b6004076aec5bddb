"""Oracles for the Pannotia applications of Table 1 -- color,
mis and p-sssp -- ported to cooperative kernels (TEST INFRASTRUCTURE ONLY: only
tests/, __graft_entry__.smoke() and bench.py may import this module).

The paper names the applications and their barrier counts (color 2/2, mis 3/3,
p-sssp 3/3 resizing barriers) but not their code (Pannotia's);
DESIGN.md reading R23 fixes the algorithms:

* color  -- Jones-Plassmann with fixed priorities: in iteration c every
            uncoloured vertex whose priority exceeds that of every neighbour
            uncoloured at the start of the iteration takes colour c.
* mis    -- Luby's maximal independent set with fixed priorities: in iteration
            t every undecided vertex whose priority is below that of every
            undecided neighbour joins the set; then every undecided neighbour
            of a member leaves.
* p-sssp -- Bellman-Ford over all vertices each iteration (Pannotia's sssp is
            not worklist-driven): dist'(v) = min(dist(v), min_u dist(u) + w(u,v)),
            until no distance changes.

Priorities are the counter-based generator both sides implement: prio(v) =
(splitmix64(seed ^ v), v) compared lexicographically (distinct for distinct v).
The functions follow those iterations step by step; they are pinned in
tests/test_oracle_pannotia.py against independent characterisations (the
sequential greedy MIS in priority order, proper colouring, Dijkstra, closed
forms on complete graphs, stars and paths).
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
UNCOLORED = -1
UNDECIDED, IN_SET, OUT_SET = 0, 1, 2
INF = 0xFFFFFFFF


def splitmix64(x: int) -> int:
    """The published splitmix64 finaliser (Steele, Lea, Flood 2014)."""
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def priorities(V: int, seed: int) -> list[tuple[int, int]]:
    return [(splitmix64((seed ^ v) & M64), v) for v in range(V)]


def color(ro, col, V: int, seed: int) -> tuple[np.ndarray, int]:
    """Jones-Plassmann colouring; returns (colour per vertex, iterations)."""
    pr = priorities(V, seed)
    c = [UNCOLORED] * V
    it = 0
    while any(x == UNCOLORED for x in c):
        start = list(c)                           # state at the start of the iteration
        for v in range(V):
            if start[v] != UNCOLORED:
                continue
            if all(pr[v] > pr[u] for u in col[ro[v]:ro[v + 1]] if start[u] == UNCOLORED):
                c[v] = it
        it += 1
    return np.array(c, dtype=np.int32), it


def mis(ro, col, V: int, seed: int) -> tuple[np.ndarray, int]:
    """Luby's MIS with fixed priorities; returns (state per vertex: 1 in, 2 out), iterations."""
    pr = priorities(V, seed)
    s = [UNDECIDED] * V
    it = 0
    while any(x == UNDECIDED for x in s):
        start = list(s)
        for v in range(V):                        # join: local minimum among undecided neighbours
            if start[v] == UNDECIDED and all(pr[v] < pr[u] for u in col[ro[v]:ro[v + 1]]
                                             if start[u] == UNDECIDED):
                s[v] = IN_SET
        mid = list(s)
        for v in range(V):                        # leave: a neighbour joined
            if mid[v] == UNDECIDED and any(mid[u] == IN_SET for u in col[ro[v]:ro[v + 1]]):
                s[v] = OUT_SET
        it += 1
    return np.array(s, dtype=np.int32), it


def p_sssp(ro, col, w, V: int, source: int) -> tuple[np.ndarray, int]:
    """Bellman-Ford over all vertices (pull form); returns (dist u32, iterations)."""
    d = [INF] * V
    d[source] = 0
    it = 0
    while True:
        nd = list(d)
        for v in range(V):
            for e in range(ro[v], ro[v + 1]):
                u = col[e]
                if d[u] != INF and d[u] + w[e] < nd[v]:
                    nd[v] = d[u] + w[e]
        it += 1
        if nd == d:
            return np.array(d, dtype=np.uint32), it
        d = nd


def greedy_mis(ro, col, V: int, seed: int) -> np.ndarray:
    """Sequential greedy MIS in increasing priority order (an independent characterisation)."""
    pr = priorities(V, seed)
    s = [UNDECIDED] * V
    for _, v in sorted(pr):
        if s[v] == UNDECIDED:
            s[v] = IN_SET
            for u in col[ro[v]:ro[v + 1]]:
                if s[u] == UNDECIDED:
                    s[u] = OUT_SET
    return np.array(s, dtype=np.int32)
