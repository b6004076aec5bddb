"""CPU tests of the partitioned path's host logic: partition layout, per-rank
generation, hub selection, the IPC-handle all-gather, and the per-level exchange
protocol of the partitioned BFS over torch.distributed (gloo, world_size 2, 127.0.0.1)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import graphgen as gg
from oracle import partition_sim as ps
from oracle import textbook as tb


def test_part_bounds_are_word_aligned_and_cover():
    for V, P in [(1, 1), (31, 2), (1000, 3), (1 << 16, 8), (100, 8)]:
        b = gg.part_bounds(V, P)
        assert b[0] == 0 and b[-1] == V and len(b) == P + 1
        assert all(x % 32 == 0 or x == V for x in b[:-1])      # empty trailing ranks start at V
        nw = (V + 31) // 32
        sw = (nw + P - 1) // P                                  # uniform slices (in-place all-gather)
        assert all(b[q] == min(V, 32 * sw * q) for q in range(P))
        assert all(b[i] <= b[i + 1] for i in range(P))


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_partition_keeps_exactly_owned_destinations(P):
    g = gg.rmat(10, seed=5)
    ro, col = g.row_offsets.numpy(), g.col_idx.numpy()
    total = 0
    for r in range(P):
        p = gg.partition(g, P, r)
        lro, lcol = p.row_offsets.numpy(), p.col_local.numpy()
        for u in range(0, g.num_vertices, 37):
            full = col[ro[u]:ro[u + 1]]
            own = full[(full >= p.v_begin) & (full < p.v_end)] - p.v_begin
            np.testing.assert_array_equal(lcol[lro[u]:lro[u + 1]], own)
        total += p.num_edges
    assert total == g.num_edges


@pytest.mark.parametrize("P", [2, 3])
def test_rmat_partition_equals_partition_of_rmat(P):
    g = gg.rmat(10, seed=7)
    for r in range(P):
        a = gg.partition(g, P, r)
        b = gg.rmat_partition(10, P, r, seed=7, chunk=3000)
        assert torch.equal(a.row_offsets, b.row_offsets) and torch.equal(a.col_local, b.col_local)


def test_hubs_of():
    from paper_1707_01989_b200 import partitioned as pt
    g = gg.disjoint_union(gg.star(5000), gg.path(10))
    p = gg.partition(g, 2, 0)
    ids, pref = pt.hubs_of(p, hub_degree=1000)
    ld = p.local_degrees()
    assert ids.tolist() == torch.nonzero(ld >= 1000).flatten().tolist()
    assert pref[-1].item() == int(ld[ld >= 1000].sum())


def test_partition_sim_uses_any_boundaries():
    """BFS levels do not depend on the partition boundaries (oracle O5 vs O1)."""
    g = gg.rmat(9, seed=1)
    s = gg.sample_sources(g, 1)[0]
    lv, _ = ps.bfs_partitioned(g.row_offsets.numpy(), g.col_idx.numpy().astype(np.int64), g.num_vertices, s, 5)
    np.testing.assert_array_equal(lv, tb.bfs(g, s))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1707_01989_b200 import partitioned as pt
    blob = bytes([rank]) * 128                      # stands in for two 64-byte IPC handles
    allh = pt.exchange_handles(blob)
    q.put((rank, [h[:1] for h in allh], [len(h) for h in allh]))
    dist.destroy_process_group()


def test_exchange_handles_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, heads, lens in res:
        assert heads == [b"\x00", b"\x01"] and lens == [128, 128]


def _bfs_worker(rank, world, port, q):
    """One rank of the NCCL data plane's protocol (coop_bfs_part_nccl), with the
    collective done by gloo and the rank-local expansion written plainly: uniform slices of the
    frontier bitmap (graphgen.part_bounds), per level an all-gather of the own slice and of the
    rank's discovered count, termination when every gathered count is 0."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = gg.rmat(10, seed=5)
    V = g.num_vertices
    s = gg.sample_sources(g, 1)[0]
    p = gg.partition(g, world, rank)
    vb, ve = p.v_begin, p.v_end
    lro, lcol = p.row_offsets.numpy().astype(np.int64), p.col_local.numpy().astype(np.int64)
    nw = (V + 31) // 32
    sw = (nw + world - 1) // world
    assert vb == min(V, 32 * sw * rank)                     # the rank's slice is words [rank*sw, (rank+1)*sw)
    F = np.zeros(world * sw, dtype=np.uint64)
    F[s >> 5] |= np.uint64(1) << np.uint64(s & 31)
    lv = np.full(ve - vb, -1, dtype=np.int64)
    if vb <= s < ve:
        lv[s - vb] = 0
    L = 0
    while True:
        mine = np.zeros(sw, dtype=np.uint64)
        words = np.nonzero(F)[0]
        cnt = 0
        for w in words:
            bits = int(F[w])
            while bits:
                b = (bits & -bits).bit_length() - 1
                bits &= bits - 1
                u = 32 * int(w) + b
                for j in range(lro[u], lro[u + 1]):
                    v = lcol[j]
                    if lv[v] < 0:
                        lv[v] = L + 1
                        gv = vb + v
                        mine[(gv >> 5) - rank * sw] |= np.uint64(1) << np.uint64(gv & 31)
                        cnt += 1
        slices = [torch.zeros(sw, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(slices, torch.from_numpy(mine.astype(np.int64)))
        counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(counts, torch.tensor([cnt], dtype=torch.int64))
        F = np.concatenate([t.numpy() for t in slices]).astype(np.uint64)
        if sum(int(c.item()) for c in counts) == 0:
            break
        L += 1
    q.put((rank, vb, lv.tolist(), L))
    dist.destroy_process_group()


def test_partitioned_bfs_protocol_gloo_world2():
    """The per-level exchange of the partitioned BFS (slice layout, counts, termination) across two
    OS processes over torch.distributed (gloo): the gathered levels equal O1's, and both ranks stop at
    the same level."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bfs_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    g = gg.rmat(10, seed=5)
    s = gg.sample_sources(g, 1)[0]
    ref = tb.bfs(g, s)
    lv = np.concatenate([np.array(r[2], dtype=np.int64) for r in res])
    np.testing.assert_array_equal(lv, ref)
    assert res[0][3] == res[1][3] == int(ref.max())          # the last level expands to nothing on both
