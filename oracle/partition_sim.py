"""O5: 1-D vertex-partitioned level-synchronous BFS (TEST INFRASTRUCTURE ONLY).

Not in the paper (single iGPU); BASELINE.json north_star / SURVEY §8(e).
P ranks are plain loops; the per-level frontier all-gather is a concatenation
of the ranks' owned next-frontier bitmaps.  Rank p owns vertices
[v_begin(p), v_end(p)) with v_begin(p) = floor(p*V/P) and stores every edge
(u, v) whose destination v it owns.  Each level every rank expands the whole
global frontier over its local edges and claims only owned vertices.
"""
from __future__ import annotations

import numpy as np


def owner_range(V: int, P: int, p: int) -> tuple[int, int]:
    return (p * V) // P, ((p + 1) * V) // P


def partition(ro: np.ndarray, col: np.ndarray, V: int, P: int):
    """Per rank: (v_begin, v_end, local_ro[V+1], local_col (global ids, owned))."""
    src = np.repeat(np.arange(V, dtype=np.int64), np.diff(ro))
    parts = []
    for p in range(P):
        b, e = owner_range(V, P, p)
        keep = (col >= b) & (col < e)
        s, d = src[keep], col[keep]
        lro = np.zeros(V + 1, dtype=np.int64)
        np.add.at(lro, s + 1, 1)
        lro = np.cumsum(lro)
        parts.append((b, e, lro, d.astype(np.int64)))
    return parts


def bfs_partitioned(ro: np.ndarray, col: np.ndarray, V: int, source: int, P: int):
    """Returns (levels int32[V] with -1 unreachable, per-level frontier sizes)."""
    parts = partition(ro, col, V, P)
    owned_levels = [np.full(e - b, -1, dtype=np.int32) for (b, e, _, _) in parts]
    frontier = np.zeros(V, dtype=bool)
    frontier[source] = True
    for p, (b, e, _, _) in enumerate(parts):
        if b <= source < e:
            owned_levels[p][source - b] = 0
    sizes = []
    level = 0
    while frontier.any():
        sizes.append(int(frontier.sum()))
        nxt_parts = []
        fverts = np.nonzero(frontier)[0]
        for p, (b, e, lro, lcol) in enumerate(parts):
            nxt = np.zeros(e - b, dtype=bool)
            for u in fverts:
                for v in lcol[lro[u]:lro[u + 1]]:
                    if owned_levels[p][v - b] == -1:
                        owned_levels[p][v - b] = level + 1
                        nxt[v - b] = True
            nxt_parts.append(nxt)
        frontier = np.concatenate(nxt_parts)          # the all-gather
        level += 1
    return np.concatenate(owned_levels), sizes
