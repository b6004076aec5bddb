"""Pins for O1 (oracle/textbook.c): closed forms, special cases and a library
routine (scipy.sparse.csgraph), never the oracle's own code."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.csgraph as csg

import graphgen as gg
from oracle import textbook as tb


def _scipy_matrix(g, weighted):
    ro = g.row_offsets.numpy()
    col = g.col_idx.numpy()
    data = g.weights.numpy().astype(np.float64) if weighted else np.ones(col.size)
    return sp.csr_matrix((data, col, ro), shape=(g.num_vertices, g.num_vertices))


@pytest.mark.parametrize("R,C,r0,c0", [(8, 8, 0, 0), (8, 8, 3, 5), (5, 13, 4, 12), (1, 9, 0, 4), (32, 7, 16, 3)])
def test_bfs_grid_closed_form(R, C, r0, c0):
    g = gg.grid(R, C)
    lv = tb.bfs(g, r0 * C + c0)
    r, c = np.divmod(np.arange(R * C), C)
    np.testing.assert_array_equal(lv, np.abs(r - r0) + np.abs(c - c0))


def test_bfs_c1_level_sizes():
    lv = tb.bfs(gg.grid(8, 8), 0)
    assert tb.level_sizes(lv) == [1, 2, 3, 4, 5, 6, 7, 8, 7, 6, 5, 4, 3, 2, 1]


def test_bfs_path_star_tree_disconnected():
    np.testing.assert_array_equal(tb.bfs(gg.path(5), 0), [0, 1, 2, 3, 4])
    lv = tb.bfs(gg.path(1000), 0)
    assert lv.max() == 999 and len(tb.level_sizes(lv)) == 1000
    np.testing.assert_array_equal(tb.bfs(gg.path(9), 4), np.abs(np.arange(9) - 4))
    s = tb.bfs(gg.star(1000), 0)
    assert s[0] == 0 and (s[1:] == 1).all()
    leaf = tb.bfs(gg.star(10), 7)
    np.testing.assert_array_equal(leaf, [1, 2, 2, 2, 2, 2, 2, 0, 2, 2])
    bt = tb.bfs(gg.binary_tree(6), 0)
    np.testing.assert_array_equal(bt, np.floor(np.log2(np.arange(1, 128))).astype(int))
    u = gg.disjoint_union(gg.path(4), gg.path(3))
    np.testing.assert_array_equal(tb.bfs(u, 1), [1, 0, 1, 2, -1, -1, -1])
    e = tb.bfs(gg.empty(5), 2)
    np.testing.assert_array_equal(e, [-1, -1, 0, -1, -1])


def test_bfs_rejects_bad_source():
    with pytest.raises(ValueError):
        tb.bfs(gg.path(3), 3)
    with pytest.raises(ValueError):
        tb.bfs(gg.path(3), -1)


@pytest.mark.parametrize("scale", [8, 10, 12])
def test_bfs_matches_scipy_on_rmat(scale):
    g = gg.rmat(scale, seed=scale)
    A = _scipy_matrix(g, weighted=False)
    for s in gg.sample_sources(g, 4):
        ref = csg.shortest_path(A, method="D", unweighted=True, indices=s)
        ref = np.where(np.isinf(ref), -1, ref).astype(np.int32)
        np.testing.assert_array_equal(tb.bfs(g, s), ref)


def test_dijkstra_unit_and_constant_weights_reduce_to_bfs():
    for g in [gg.grid(17, 23), gg.rmat(10, seed=3), gg.disjoint_union(gg.grid(4, 4), gg.path(5))]:
        lv = tb.bfs(g, 0).astype(np.int64)
        for c in (1, 7, 1000):
            d = tb.dijkstra(gg.with_constant_weights(g, c), 0).astype(np.int64)
            np.testing.assert_array_equal(d, np.where(lv < 0, 0xFFFFFFFF, lv * c))


def test_dijkstra_path_prefix_sums():
    g = gg.with_weights(gg.path(50), seed=9)
    w = g.weights.numpy()
    # edge i-(i+1): weight of the directed edge from i to i+1
    step = np.array([w[g.row_offsets[i]: g.row_offsets[i + 1]][g.col_idx[g.row_offsets[i]: g.row_offsets[i + 1]].numpy() == i + 1][0]
                     for i in range(49)])
    d = tb.dijkstra(g, 0)
    np.testing.assert_array_equal(d, np.concatenate([[0], np.cumsum(step)]))


@pytest.mark.parametrize("mk", [lambda: gg.with_weights(gg.grid(30, 40), seed=1),
                                lambda: gg.with_weights(gg.rmat(11, seed=5), seed=2),
                                lambda: gg.with_weights(gg.disjoint_union(gg.rmat(8), gg.grid(5, 5)), seed=3)])
def test_dijkstra_matches_scipy(mk):
    g = mk()
    A = _scipy_matrix(g, weighted=True)
    for s in [0] + gg.sample_sources(g, 3):
        ref = csg.dijkstra(A, indices=s)
        ref = np.where(np.isinf(ref), 0xFFFFFFFF, ref).astype(np.uint64)
        np.testing.assert_array_equal(tb.dijkstra(g, s).astype(np.uint64), ref)
