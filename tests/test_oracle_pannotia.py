"""Pins for oracle/pannotia.py (color, mis, p-sssp of Table 1):
the round-based oracles against independent characterisations -- the sequential
greedy MIS in priority order (Luby with fixed priorities computes exactly it),
independence + maximality, proper colouring, closed forms on complete graphs and
stars, splitmix64's published outputs, and Dijkstra for p-sssp."""
import numpy as np
import pytest
import torch

import graphgen as gg
from oracle import pannotia as pn
from oracle import textbook as tb


def _arrs(g):
    return g.row_offsets.tolist(), g.col_idx.tolist()


def complete(n):
    src = torch.tensor([u for u in range(n) for v in range(n) if u != v])
    dst = torch.tensor([v for u in range(n) for v in range(n) if u != v])
    return gg.edges_to_csr(src, dst, n)


def test_splitmix64_published_outputs():
    # splitmix64 with state 0: first outputs of the published generator (state += golden, mix)
    assert pn.splitmix64(0) == 0xE220A8397B1DCDAF
    assert pn.splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


GRAPHS = {"rmat9": lambda: gg.rmat(9, seed=4), "grid": lambda: gg.grid(13, 9), "star": lambda: gg.star(40),
          "path": lambda: gg.path(50), "disconnected": lambda: gg.disjoint_union(gg.rmat(7, seed=2), gg.path(9))}


@pytest.mark.parametrize("name", sorted(GRAPHS))
@pytest.mark.parametrize("seed", [1, 7])
def test_mis_equals_greedy_in_priority_order(name, seed):
    g = GRAPHS[name]()
    ro, col = _arrs(g)
    V = g.num_vertices
    s, _ = pn.mis(ro, col, V, seed)
    np.testing.assert_array_equal(s, pn.greedy_mis(ro, col, V, seed))
    inset = s == pn.IN_SET
    for v in range(V):
        nb = col[ro[v]:ro[v + 1]]
        if inset[v]:
            assert not any(inset[u] for u in nb)                  # independent
        else:
            assert s[v] == pn.OUT_SET and any(inset[u] for u in nb)   # maximal


@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_color_is_proper_and_complete(name):
    g = GRAPHS[name]()
    ro, col = _arrs(g)
    c, iters = pn.color(ro, col, g.num_vertices, 3)
    assert (c >= 0).all() and c.max() == iters - 1
    for v in range(g.num_vertices):
        assert all(c[u] != c[v] for u in col[ro[v]:ro[v + 1]])


def test_color_closed_forms():
    # K_n: one vertex per iteration, in decreasing priority
    n = 7
    g = complete(n)
    ro, col = _arrs(g)
    c, iters = pn.color(ro, col, n, 5)
    pr = pn.priorities(n, 5)
    order = [v for _, v in sorted(pr, reverse=True)]
    assert [int(c[v]) for v in order] == list(range(n)) and iters == n
    # star: leaves above the centre take colour 0; the centre takes 0 if it beats every leaf,
    # else 1; the leaves below it take 1 (centre at 0) or 2 (centre at 1)
    g = gg.star(30)
    ro, col = _arrs(g)
    for seed in (1, 2, 3, 11):
        c, _ = pn.color(ro, col, 30, seed)
        pr = pn.priorities(30, seed)
        top = all(pr[0] > pr[v] for v in range(1, 30))
        assert c[0] == (0 if top else 1)
        for v in range(1, 30):
            assert c[v] == (0 if pr[v] > pr[0] else (1 if top else 2))


def test_mis_closed_forms():
    g = complete(6)
    ro, col = _arrs(g)
    s, iters = pn.mis(ro, col, 6, 9)
    pr = pn.priorities(6, 9)
    assert [v for v in range(6) if s[v] == pn.IN_SET] == [min(pr)[1]] and iters == 1


@pytest.mark.parametrize("name", ["grid", "rmat9", "disconnected"])
def test_p_sssp_equals_dijkstra(name):
    g = gg.with_weights(GRAPHS[name](), seed=2)
    ro, col = _arrs(g)
    w = [int(x) for x in g.weights.tolist()]
    for s in gg.sample_sources(g, 2):
        d, _ = pn.p_sssp(ro, col, w, g.num_vertices, s)
        np.testing.assert_array_equal(d, tb.dijkstra(g, s))
