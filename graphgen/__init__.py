"""Seeded synthetic graph generators (input data only).

This module is the ONE piece of code shared by the oracle tests and the CUDA
path: it produces CSR graphs and seeded random draws, and contains none of the
method's arithmetic (no BFS, no relaxation, no barrier logic).  Both sides
consume the *arrays* it returns.

The paper names its inputs only ("USA road", "G3_circuit", "rmat";
PAPER.md:1110, :1195-1198, :1224) and ships no datasets, so the shapes follow
SURVEY.md §8(c) "Generator definitions" and §8(d):

* ``grid(R, C)``   -- 2-D 4-neighbour grid, id = r*C + c (road-network shape:
  deep, many levels, small frontiers).
* ``rmat(scale)``  -- Graph500-parameterised R-MAT (a,b,c,d = .57,.19,.19,.05,
  edgefactor 16), seeded random relabel, symmetrised, self-loops dropped,
  duplicates merged (wide, few levels, huge frontiers).
* ``path``, ``star``, ``binary_tree``, ``disjoint_union`` -- closed-form shapes.
* ``pair_weights`` -- integer weight per undirected pair, uniform in [1, wmax].

All randomness is counter-based (splitmix64 over int64 tensors), so a graph is
bit-identical on CPU and CUDA for the same seed.  Every function is
device-agnostic: pass ``device="cuda"`` to generate large graphs on the GPU.
"""
from __future__ import annotations

import dataclasses
import hashlib
from typing import Optional

import torch

__all__ = [
    "CSR", "splitmix64", "uniform_u53", "edges_to_csr", "grid", "path", "star",
    "binary_tree", "disjoint_union", "empty", "rmat", "pair_weights",
    "sample_sources", "graph_hash",
]

_M64 = (1 << 64) - 1


def _s64(c: int) -> int:
    """Unsigned 64-bit constant -> the int64 with the same bit pattern."""
    c &= _M64
    return c - (1 << 64) if c >= (1 << 63) else c


_GOLDEN = _s64(0x9E3779B97F4A7C15)
_MIX1 = _s64(0xBF58476D1CE4E5B9)
_MIX2 = _s64(0x94D049BB133111EB)


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (two's-complement wraparound)."""
    z = x + _GOLDEN
    z = (z ^ _srl(z, 30)) * _MIX1
    z = (z ^ _srl(z, 27)) * _MIX2
    return z ^ _srl(z, 31)


def splitmix64_int(x: int) -> int:
    """Scalar splitmix64 on Python ints (same function as :func:`splitmix64`)."""
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def uniform_u53(z: torch.Tensor) -> torch.Tensor:
    """Top 53 bits of a 64-bit hash as a non-negative int64 in [0, 2^53)."""
    return _srl(z, 11)


@dataclasses.dataclass
class CSR:
    """Compressed sparse rows; neighbour lists sorted ascending.

    row_offsets: int64[V+1]; col_idx: int32[E]; weights: int32[E] or None
    (values in [1, wmax], read as uint32 by the CUDA path).
    """

    num_vertices: int
    row_offsets: torch.Tensor
    col_idx: torch.Tensor
    weights: Optional[torch.Tensor] = None
    name: str = ""

    @property
    def num_edges(self) -> int:
        return int(self.col_idx.numel())

    def to(self, device) -> "CSR":
        w = None if self.weights is None else self.weights.to(device)
        return CSR(self.num_vertices, self.row_offsets.to(device), self.col_idx.to(device), w, self.name)

    def degrees(self) -> torch.Tensor:
        return self.row_offsets[1:] - self.row_offsets[:-1]


def edges_to_csr(src: torch.Tensor, dst: torch.Tensor, num_vertices: int, *,
                 symmetrize: bool = True, name: str = "") -> CSR:
    """Edge list -> CSR: optionally symmetrise, drop self loops, merge duplicates,
    sort neighbour lists ascending (SURVEY §8(c) reading 11)."""
    src = src.to(torch.int64)
    dst = dst.to(torch.int64)
    if symmetrize:
        src, dst = torch.cat([src, dst]), torch.cat([dst, src])
    keep = src != dst
    key = src[keep] * num_vertices + dst[keep]
    del src, dst, keep
    key = torch.unique(key, sorted=True)
    s = key // num_vertices
    col = (key - s * num_vertices).to(torch.int32)
    del key
    counts = torch.bincount(s, minlength=num_vertices)
    del s
    ro = torch.zeros(num_vertices + 1, dtype=torch.int64, device=col.device)
    ro[1:] = torch.cumsum(counts, 0)
    return CSR(num_vertices, ro, col, None, name)


def empty(n: int, device="cpu") -> CSR:
    """n isolated vertices, no edges."""
    return CSR(n, torch.zeros(n + 1, dtype=torch.int64, device=device),
               torch.zeros(0, dtype=torch.int32, device=device), None, f"empty{n}")


def grid(R: int, C: int, device="cpu") -> CSR:
    """R x C 4-neighbour grid, id = r*C + c, undirected."""
    v = torch.arange(R * C, dtype=torch.int64, device=device)
    r, c = v // C, v % C
    right = v[c < C - 1]
    down = v[r < R - 1]
    src = torch.cat([right, down])
    dst = torch.cat([right + 1, down + C])
    return edges_to_csr(src, dst, R * C, name=f"grid{R}x{C}")


def path(n: int, device="cpu") -> CSR:
    """Path 0-1-2-...-(n-1)."""
    v = torch.arange(max(n - 1, 0), dtype=torch.int64, device=device)
    return edges_to_csr(v, v + 1, n, name=f"path{n}")


def star(n: int, device="cpu") -> CSR:
    """Centre 0 joined to leaves 1..n-1."""
    leaves = torch.arange(1, n, dtype=torch.int64, device=device)
    return edges_to_csr(torch.zeros_like(leaves), leaves, n, name=f"star{n}")


def binary_tree(depth: int, device="cpu") -> CSR:
    """Complete binary tree with 2^(depth+1)-1 vertices; parent(i) = (i-1)//2."""
    n = (1 << (depth + 1)) - 1
    ch = torch.arange(1, n, dtype=torch.int64, device=device)
    return edges_to_csr((ch - 1) // 2, ch, n, name=f"btree{depth}")


def disjoint_union(a: CSR, b: CSR) -> CSR:
    """Vertices of b are shifted by a.num_vertices."""
    ro = torch.cat([a.row_offsets, b.row_offsets[1:] + a.row_offsets[-1]])
    col = torch.cat([a.col_idx, b.col_idx + a.num_vertices])
    return CSR(a.num_vertices + b.num_vertices, ro, col, None, f"{a.name}+{b.name}")


def rmat(scale: int, edgefactor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
         seed: int = 1, relabel: bool = True, device="cpu", chunk: int = 1 << 25) -> CSR:
    """R-MAT / Kronecker generator with Graph500 parameters (SURVEY §8(c) reading 13).

    Tuple i, bit k draws x = top53(splitmix64((i<<6 | k) XOR splitmix64(seed)));
    quadrant by cumulative thresholds (a, a+b, a+b+c) * 2^53 (integer compare,
    device independent).  u = 2u + qu, v = 2v + qv.  A seeded random permutation
    (argsort of splitmix64 keys) relabels vertices.  NOT Graph500 bit-compatible
    (different RNG); parameters match.
    """
    V = 1 << scale
    ntup = edgefactor * V
    t1 = int(a * (1 << 53))
    t2 = int((a + b) * (1 << 53))
    t3 = int((a + b + c) * (1 << 53))
    smix = _s64(splitmix64_int(seed & _M64))
    us, vs = [], []
    for start in range(0, ntup, chunk):
        i = torch.arange(start, min(ntup, start + chunk), dtype=torch.int64, device=device)
        u = torch.zeros_like(i)
        v = torch.zeros_like(i)
        base = (i << 6) ^ smix
        del i
        for k in range(scale):
            x = uniform_u53(splitmix64(base ^ k))
            qu = (x >= t2).to(torch.int64)                     # quadrants c, d -> lower half
            qv = ((x >= t1) & (x < t2)) | (x >= t3)            # quadrants b, d -> right half
            u = (u << 1) | qu
            v = (v << 1) | qv.to(torch.int64)
            del x, qu, qv
        us.append(u)
        vs.append(v)
        del base
    u = torch.cat(us)
    v = torch.cat(vs)
    del us, vs
    if relabel:
        perm_keys = splitmix64(torch.arange(V, dtype=torch.int64, device=device) ^ _s64(splitmix64_int((seed + 0x5EED) & _M64)))
        order = torch.argsort(perm_keys, stable=True)      # order[j] = old id placed at new id j
        pi = torch.empty_like(order)
        pi[order] = torch.arange(V, dtype=torch.int64, device=device)   # pi[old] = new
        u = pi[u]
        v = pi[v]
        del pi, order, perm_keys
    g = edges_to_csr(u, v, V, name=f"rmat{scale}")
    return g


def pair_weights(g: CSR, seed: int = 1, wmax: int = 1000) -> torch.Tensor:
    """Weight of directed edge (u,v) = 1 + ((splitmix64(s ^ (min<<32 | max)) >>> 33) mod wmax).

    Symmetric by construction (both directions of a pair get the same weight).
    Returned as int32 in [1, wmax] (read as uint32 by the CUDA path).
    """
    V = g.num_vertices
    deg = g.degrees()
    src = torch.repeat_interleave(torch.arange(V, dtype=torch.int64, device=g.col_idx.device), deg)
    dst = g.col_idx.to(torch.int64)
    lo = torch.minimum(src, dst)
    hi = torch.maximum(src, dst)
    z = splitmix64(((lo << 32) | hi) ^ _s64(splitmix64_int((seed * 0x2545F4914F6CDD1D) & _M64)))
    return (1 + (_srl(z, 33) % wmax)).to(torch.int32)


def with_weights(g: CSR, seed: int = 1, wmax: int = 1000) -> CSR:
    return CSR(g.num_vertices, g.row_offsets, g.col_idx, pair_weights(g, seed, wmax), g.name + f"_w{wmax}")


def with_constant_weights(g: CSR, c: int) -> CSR:
    return CSR(g.num_vertices, g.row_offsets, g.col_idx,
               torch.full_like(g.col_idx, c, dtype=torch.int32), g.name + f"_c{c}")


def sample_sources(g: CSR, count: int, seed: int = 2) -> list[int]:
    """`count` distinct vertices with degree > 0, chosen by seeded hash order."""
    deg = g.degrees().cpu()
    cand = torch.nonzero(deg > 0).flatten()
    if cand.numel() == 0:
        return [0] * min(count, 1)
    keys = splitmix64(cand ^ _s64(splitmix64_int((seed + 0xB5) & _M64)))
    order = torch.argsort(keys, stable=True)
    return [int(x) for x in cand[order[:count]]]


def graph_hash(g: CSR) -> str:
    """Content hash of the CSR arrays (sha256, first 16 hex digits)."""
    h = hashlib.sha256()
    h.update(str(g.num_vertices).encode())
    h.update(g.row_offsets.cpu().numpy().tobytes())
    h.update(g.col_idx.cpu().numpy().tobytes())
    if g.weights is not None:
        h.update(g.weights.cpu().numpy().tobytes())
    return h.hexdigest()[:16]


# ---------------------------------------------------------------- 1-D partition (configs[4])
@dataclasses.dataclass
class PartCSR:
    """Rank `rank`'s share of a 1-D vertex partition: every edge (u, v) whose
    destination v lies in [v_begin, v_end), indexed by the GLOBAL source u
    (row_offsets has V+1 entries), destinations stored rank-local (v - v_begin)."""
    num_vertices: int
    v_begin: int
    v_end: int
    rank: int
    nranks: int
    row_offsets: torch.Tensor
    col_local: torch.Tensor
    weights: Optional[torch.Tensor] = None     # of the local edges (weighted graphs)

    @property
    def num_edges(self) -> int:
        return int(self.col_local.numel())

    def local_degrees(self) -> torch.Tensor:
        return self.row_offsets[1:] - self.row_offsets[:-1]


def part_rows(part: PartCSR) -> tuple[torch.Tensor, torch.Tensor]:
    """Owned ROWS of a symmetric graph from its column partition: the neighbour
    list of owned vertex v (global ids, ascending) = the sources of the local edges
    pointing to v.  Returns (row_offsets int64[v_end - v_begin + 1], col int32)."""
    V = part.num_vertices
    nown = part.v_end - part.v_begin
    dev = part.col_local.device
    src = torch.repeat_interleave(torch.arange(V, dtype=torch.int64, device=dev), part.local_degrees())
    dst = part.col_local.to(torch.int64)
    key = torch.sort(dst * V + src).values
    del src
    rcol = (key % V).to(torch.int32)
    counts = torch.bincount(dst, minlength=nown)
    del key, dst
    rro = torch.zeros(nown + 1, dtype=torch.int64, device=dev)
    rro[1:] = torch.cumsum(counts, 0)
    return rro, rcol


def part_bounds(V: int, P: int) -> list[int]:
    """Owned-range boundaries: uniform slices of sw = ceil(ceil(V/32) / P) bitmap
    words per rank (rank p owns [32*sw*p, min(V, 32*sw*(p+1)))), so the slice
    all-gather of the frontier bitmap is one in-place NCCL all-gather."""
    nw = (V + 31) // 32
    sw = (nw + P - 1) // P
    b = [min(V, p * sw * 32) for p in range(P)]
    return b + [V]


def partition(g: CSR, P: int, rank: int) -> PartCSR:
    b = part_bounds(g.num_vertices, P)
    vb, ve = b[rank], b[rank + 1]
    col = g.col_idx
    keep = (col >= vb) & (col < ve)
    cm = torch.zeros(col.numel() + 1, dtype=torch.int64, device=col.device)
    cm[1:] = torch.cumsum(keep.to(torch.int64), 0)
    ro = cm[g.row_offsets]
    w = None if g.weights is None else g.weights[keep]
    return PartCSR(g.num_vertices, vb, ve, rank, P, ro, (col[keep] - vb).to(torch.int32), w)


def rmat_partition(scale: int, P: int, rank: int, edgefactor: int = 16, seed: int = 1, device="cpu",
                   chunk: int = 1 << 25) -> PartCSR:
    """Rank `rank`'s share of rmat(scale, ...) built without materialising the
    whole graph: the same tuples are drawn, but only the directed entries whose
    destination this rank owns are kept (equals partition(rmat(...), P, rank))."""
    V = 1 << scale
    ntup = edgefactor * V
    a, bq, c = 0.57, 0.19, 0.19
    t1, t2, t3 = int(a * (1 << 53)), int((a + bq) * (1 << 53)), int((a + bq + c) * (1 << 53))
    smix = _s64(splitmix64_int(seed & _M64))
    perm_keys = splitmix64(torch.arange(V, dtype=torch.int64, device=device) ^ _s64(splitmix64_int((seed + 0x5EED) & _M64)))
    order = torch.argsort(perm_keys, stable=True)
    pi = torch.empty_like(order)
    pi[order] = torch.arange(V, dtype=torch.int64, device=device)
    del perm_keys, order
    bnd = part_bounds(V, P)
    vb, ve = bnd[rank], bnd[rank + 1]
    keys = []
    for start in range(0, ntup, chunk):
        i = torch.arange(start, min(ntup, start + chunk), dtype=torch.int64, device=device)
        u = torch.zeros_like(i)
        v = torch.zeros_like(i)
        base = (i << 6) ^ smix
        del i
        for k in range(scale):
            x = uniform_u53(splitmix64(base ^ k))
            u = (u << 1) | (x >= t2).to(torch.int64)
            v = (v << 1) | (((x >= t1) & (x < t2)) | (x >= t3)).to(torch.int64)
            del x
        del base
        u = pi[u]
        v = pi[v]
        src = torch.cat([u, v])
        dst = torch.cat([v, u])
        del u, v
        keep = (src != dst) & (dst >= vb) & (dst < ve)
        keys.append(torch.unique(src[keep] * V + dst[keep]))
        del src, dst, keep
    key = torch.unique(torch.cat(keys)) if keys else torch.zeros(0, dtype=torch.int64, device=device)
    del keys
    s = key // V
    d = (key - s * V - vb).to(torch.int32)
    del key
    counts = torch.bincount(s, minlength=V)
    ro = torch.zeros(V + 1, dtype=torch.int64, device=device)
    ro[1:] = torch.cumsum(counts, 0)
    return PartCSR(V, vb, ve, rank, P, ro, d)
