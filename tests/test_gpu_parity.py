"""GPU parity: the CUDA path through the C ABI vs the oracle, element by
element, on seeded inputs.  Bit-exact for BFS levels and
integer SSSP distances under every kill/fork schedule."""
import numpy as np
import pytest
import torch

import graphgen as gg
from conftest import golden
from oracle import coop_sim as cs
from oracle import textbook as tb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def coop():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1707_01989_b200 import build, coop as c
    build.build()
    return c


def _dev(g):
    return g.to("cuda")


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


GRAPHS = {
    "grid8": lambda: gg.grid(8, 8),
    "grid_ragged": lambda: gg.grid(37, 53),
    "path1000": lambda: gg.path(1000),
    "star5000": lambda: gg.star(5000),
    "btree10": lambda: gg.binary_tree(10),
    "disconnected": lambda: gg.disjoint_union(gg.rmat(10, seed=3), gg.grid(9, 9)),
    "rmat12": lambda: gg.rmat(12, seed=1),
    "rmat16": lambda: gg.rmat(16, seed=1),
}


@pytest.mark.parametrize("name", list(GRAPHS))
def test_bfs_never_resize(coop, name):
    g = GRAPHS[name]()
    gd = _dev(g)
    for s in ([0] + gg.sample_sources(g, 3)):
        lv, st = coop.bfs(gd, s, level_cap=4096)
        ref = tb.bfs(g, s)
        np.testing.assert_array_equal(lv.cpu().numpy(), ref)
        assert st.levels == len(tb.level_sizes(ref))
        assert st.level_sizes == tb.level_sizes(ref)
        assert st.reached == int((ref >= 0).sum())
        deg = np.diff(g.row_offsets.numpy())
        assert st.edges_scanned == int(deg[ref >= 0].sum())      # every reached vertex expanded once


@pytest.mark.parametrize("threads", [256, 512, 1024])
@pytest.mark.parametrize("N", [1, 3, 64])
def test_bfs_block_sizes_and_grid_sizes(coop, threads, N):
    g = gg.rmat(13, seed=9)
    gd = _dev(g)
    s = gg.sample_sources(g, 1)[0]
    lv, st = coop.bfs(gd, s, threads_per_wg=threads, max_wgs=N)
    np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(g, s))
    assert st.n_wgs == N


def test_bfs_c1_scripted_trace_matches_oracle(coop):
    """Config 1: 8x8 grid, N=4, 2 resizing barriers per level, the fixed
    kill/fork schedule; levels AND the M-per-episode trace equal the oracle's."""
    fx = golden("c1_trace.json")
    g = gg.grid(8, 8)
    script = [0] * 64
    for k, v in fx["script"].items():
        script[int(k)] = v
    sim = cs.simulate(g, 0, N=4, d=4, scheduler=cs.ScriptedScheduler({int(k): v for k, v in fx["script"].items()}, 4),
                      chooser=cs.RandomChooser(0))
    for threads in (256, 512):
        lv, st = coop.bfs(_dev(g), 0, max_wgs=4, threads_per_wg=threads, barriers_per_level=2,
                          policy=coop.POLICY_SCRIPTED, script=script, flags=coop.FLAG_CHECK, trace_cap=64,
                          level_cap=64)
        np.testing.assert_array_equal(lv.cpu().numpy(), sim.values)
        assert st.m_trace == sim.m_trace == fx["m_after_episode"]
        assert (st.kills, st.forks) == (fx["kills"], fx["forks"])
        assert st.level_sizes == fx["level_sizes"]
        assert st.episodes == 30


@pytest.mark.parametrize("bpl", [1, 2])
def test_bfs_random_resize_schedules(coop, bpl):
    for name in ["grid_ragged", "rmat12", "btree10", "disconnected"]:
        g = GRAPHS[name]()
        gd = _dev(g)
        s = gg.sample_sources(g, 1)[0]
        ref = tb.bfs(g, s)
        for seed in range(4):
            lv, st = coop.bfs(gd, s, max_wgs=40, init_wgs=1 + 7 * seed, threads_per_wg=256, barriers_per_level=bpl,
                              policy=coop.POLICY_RANDOM, resize_prob=0.7, seed=seed, flags=coop.FLAG_CHECK,
                              trace_cap=1 << 14)
            np.testing.assert_array_equal(lv.cpu().numpy(), ref)
            assert st.kills + st.forks > 0
            assert all(1 <= m <= 40 for m in st.m_trace)


@pytest.mark.parametrize("flags", [0, "diropt"])
def test_bfs_plain_noncoop_baseline(coop, flags):
    """The separately compiled non-cooperative kernel (kCoop=false, selected by BARRIER_PLAIN)."""
    g = gg.rmat(14, seed=4)
    fl = coop.FLAG_DIROPT if flags else 0
    for s in gg.sample_sources(g, 3):
        for thr in (256, 512, 1024):
            lv, st = coop.bfs(_dev(g), s, barrier_mode=coop.BARRIER_PLAIN, threads_per_wg=thr, flags=fl)
            np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(g, s))
            assert st.kills == 0 and st.forks == 0


def test_sssp_plain_noncoop_baseline(coop):
    g = gg.with_weights(gg.grid(40, 31), seed=5)
    for delta in (0, 3000):
        d, st = coop.sssp(_dev(g), 7, barrier_mode=coop.BARRIER_PLAIN, sssp_delta=delta)
        np.testing.assert_array_equal(_u32(d), tb.dijkstra(g, 7))


def test_bfs_edge_cases(coop):
    # single vertex, isolated source, empty graph
    lv, st = coop.bfs(_dev(gg.empty(1)), 0)
    assert lv.cpu().tolist() == [0]
    lv, _ = coop.bfs(_dev(gg.empty(37)), 5)
    assert lv.cpu().tolist() == [-1] * 5 + [0] + [-1] * 31
    g = gg.disjoint_union(gg.path(3), gg.star(4))
    lv, _ = coop.bfs(_dev(g), 4)
    np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(g, 4))
    with pytest.raises(coop.CoopError) as e:
        coop.bfs(_dev(gg.path(4)), 4)
    assert e.value.status == 1
    with pytest.raises(coop.CoopError) as e:
        coop.bfs(_dev(gg.path(4)), 0, max_wgs=100000)
    assert e.value.status in (1, 3)
    # unaligned output buffer (head/tail paths of the vectorised init)
    g = gg.grid(11, 13)
    buf = torch.empty(g.num_vertices + 3, dtype=torch.int32, device="cuda")
    lv, _ = coop.bfs(_dev(g), 7, levels_out=buf[3:])
    np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(g, 7))


def test_bfs_hub_heavy_split(coop):
    """A star with a huge centre exercises the edge-balanced heavy path."""
    g = gg.disjoint_union(gg.star(300000), gg.rmat(12, seed=2))
    gd = _dev(g)
    for s in (0, 17, 300001):
        lv, _ = coop.bfs(gd, s)
        np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(g, s))


# ---------------------------------------------------------------- SSSP
SSSP_GRAPHS = {
    "grid_w": lambda: gg.with_weights(gg.grid(64, 48), seed=1),
    "rmat_w": lambda: gg.with_weights(gg.rmat(13, seed=6), seed=2),
    "grid_c1": lambda: gg.with_constant_weights(gg.grid(40, 40), 1),
    "path_w": lambda: gg.with_weights(gg.path(3000), seed=5),
    "disc_w": lambda: gg.with_weights(gg.disjoint_union(gg.grid(20, 20), gg.rmat(9, seed=3)), seed=4),
}


@pytest.mark.parametrize("name", list(SSSP_GRAPHS))
def test_sssp_matches_dijkstra(coop, name):
    g = SSSP_GRAPHS[name]()
    gd = _dev(g)
    for s in [0] + gg.sample_sources(g, 2):
        d, st = coop.sssp(gd, s)
        np.testing.assert_array_equal(_u32(d), tb.dijkstra(g, s))


def test_sssp_unit_weights_equal_bfs(coop):
    g = gg.with_constant_weights(gg.rmat(12, seed=8), 1)
    s = gg.sample_sources(g, 1)[0]
    d, _ = coop.sssp(_dev(g), s)
    lv = tb.bfs(g, s).astype(np.int64)
    np.testing.assert_array_equal(_u32(d).astype(np.int64), np.where(lv < 0, 0xFFFFFFFF, lv))


def test_sssp_random_resize(coop):
    g = SSSP_GRAPHS["grid_w"]()
    gd = _dev(g)
    ref = tb.dijkstra(g, 5)
    for seed in range(4):
        d, st = coop.sssp(gd, 5, max_wgs=24, threads_per_wg=256, policy=coop.POLICY_RANDOM, resize_prob=0.5,
                          seed=seed, flags=coop.FLAG_CHECK)
        np.testing.assert_array_equal(_u32(d), ref)
        assert st.kills > 0


def test_sssp_overflow_rejected(coop):
    g = gg.with_constant_weights(gg.path(5_000_000), 1000)
    with pytest.raises(coop.CoopError) as e:
        coop.sssp(_dev(g), 0)
    assert e.value.status == 7


# ---------------------------------------------------------------- multitasking
def test_bfs_under_periodic_task(coop):
    """Scheduler CTA posts a task every 50 us demanding Q WGs: kills/forks
    happen, the task runs, the levels stay bit-exact."""
    g = gg.rmat(16, seed=1)
    gd = _dev(g)
    s = gg.sample_sources(g, 1)[0]
    ref = tb.bfs(g, s)
    info = coop.device_query(0, 256)
    N = info["max_coresident"] - 1
    for q in (1, N // 4, N // 2, N - 1):
        lv, st = coop.bfs(gd, s, threads_per_wg=256, policy=coop.POLICY_SCHEDULER, task_wgs=q, task_blocks=2 * q,
                          task_block_ns=20_000, task_period_ns=50_000, task_first_ns=0, event_cap=256,
                          flags=coop.FLAG_CHECK)
        np.testing.assert_array_equal(lv.cpu().numpy(), ref)
        assert st.tasks_posted >= 1
        ev = [e for e in st.task_events if e["t_first_start"]]
        assert ev and all(e["t_first_start"] >= e["t_arrive"] for e in ev)


def test_naive_barrier_under_task(coop):
    g = gg.grid(200, 200)
    gd = _dev(g)
    ref = tb.bfs(g, 0)
    lv, st = coop.bfs(gd, 0, threads_per_wg=256, max_wgs=64, barrier_mode=coop.BARRIER_NAIVE,
                      policy=coop.POLICY_SCHEDULER, task_wgs=16, task_blocks=16, task_block_ns=5_000,
                      task_period_ns=20_000, event_cap=512)
    np.testing.assert_array_equal(lv.cpu().numpy(), ref)
    assert st.kills > 0


def test_handle_api_host_channel(coop):
    g = gg.grid(300, 300)
    gd = _dev(g)
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
    h = coop.Handle("bfs", gd, 0, out, threads_per_wg=256, max_wgs=32)
    h.submit_task(8, 16, 10_000)
    h.demand(2)
    h.grant(2)
    assert h.query() >= 0
    st = h.wait(event_cap=16)
    np.testing.assert_array_equal(out.cpu().numpy(), tb.bfs(g, 0))
    with coop.Handle("bfs", gd, 0, out, threads_per_wg=256, max_wgs=32) as h2:
        with pytest.raises(coop.CoopError) as e:
            h2.submit_task(32, 1, 1)
        assert e.value.status == 5
        with pytest.raises(coop.CoopError) as e:   # the scratch belongs to the live handle
            coop.bfs(gd, 0)
        assert e.value.status == 10
    lv, _ = coop.bfs(gd, 0)                         # released by close()
    np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(g, 0))


def test_handle_api_repeated_mid_interval_demand(coop):
    """Regression for the mid-interval offer_kill deadlock: demand
    posted while CTAs are already arriving at the barrier must not leave a demanded
    non-top CTA waiting for a top id that can no longer leave.  The original bug hung
    about 1 run in 8 of this scenario; 12 runs here."""
    g = gg.grid(300, 300)
    gd = _dev(g)
    ref = tb.bfs(g, 0)
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
    for i in range(12):
        with coop.Handle("bfs", gd, 0, out, threads_per_wg=256, max_wgs=32, timeout_ns=5_000_000_000) as h:
            h.submit_task(8, 16, 10_000)
            h.demand(2 + i % 3)
            h.grant(2)
            h.wait(event_cap=16)
        np.testing.assert_array_equal(out.cpu().numpy(), ref)


# ---------------------------------------------------------------- barrier
@pytest.mark.parametrize("n", [148, 296, 592])
def test_barrier_bench_invariants(coop, n):
    r = coop.barrier_bench(n, 20000, threads=128, resize_prob=1 / 8, seed=3, check=True)
    assert r["violations"] == 0 and r["kills"] > 0 and r["forks"] > 0
    r = coop.barrier_bench(n, 20000, threads=128, plain=True, check=True)
    assert r["violations"] == 0


def test_end_to_end_host_pointers(coop):
    g = gg.rmat(12, seed=5)
    s = gg.sample_sources(g, 1)[0]
    ro = g.row_offsets.to(torch.int32).pin_memory()
    col = g.col_idx.pin_memory()
    out = torch.empty(g.num_vertices, dtype=torch.int32).pin_memory()
    coop.bfs_host(ro, col, s, out)
    np.testing.assert_array_equal(out.numpy(), tb.bfs(g, s))
    gw = gg.with_weights(gg.grid(30, 30), seed=3)
    outd = torch.empty(gw.num_vertices, dtype=torch.int32)
    coop.sssp_host(gw.row_offsets, gw.col_idx, gw.weights, 1000, 0, outd)
    np.testing.assert_array_equal(outd.numpy().view(np.uint32), tb.dijkstra(gw, 0))


# ---------------------------------------------------------------- direction optimisation
@pytest.mark.parametrize("name", ["rmat12", "rmat16", "disconnected", "grid_ragged", "star5000", "btree10"])
def test_bfs_direction_optimising(coop, name):
    g = GRAPHS[name]()
    gd = _dev(g)
    for s in [0] + gg.sample_sources(g, 3):
        ref = tb.bfs(g, s)
        lv, st = coop.bfs(gd, s, flags=coop.FLAG_DIROPT, level_cap=4096)
        np.testing.assert_array_equal(lv.cpu().numpy(), ref)
        assert st.level_sizes == tb.level_sizes(ref)
        assert st.reached == int((ref >= 0).sum())
    if name.startswith("rmat"):
        assert st.bottom_up_levels >= 1          # R-MAT's giant frontier triggers bottom-up


def test_bfs_direction_optimising_under_resizes(coop):
    g = gg.rmat(15, seed=2)
    gd = _dev(g)
    s = gg.sample_sources(g, 1)[0]
    ref = tb.bfs(g, s)
    for seed in range(3):
        lv, st = coop.bfs(gd, s, flags=coop.FLAG_DIROPT | coop.FLAG_CHECK, max_wgs=50, threads_per_wg=256,
                          policy=coop.POLICY_RANDOM, resize_prob=0.8, seed=seed, barriers_per_level=1 + seed % 2)
        np.testing.assert_array_equal(lv.cpu().numpy(), ref)
        assert st.kills + st.forks > 0 and st.bottom_up_levels >= 1
    info = coop.device_query(0, 256)
    lv, st = coop.bfs(gd, s, flags=coop.FLAG_DIROPT, threads_per_wg=256, policy=coop.POLICY_SCHEDULER,
                      task_wgs=(info["max_coresident"] - 1) // 2, task_blocks=64, task_block_ns=5_000,
                      task_period_ns=20_000, event_cap=64)
    np.testing.assert_array_equal(lv.cpu().numpy(), ref)


# ---------------------------------------------------------------- SSSP near-far
@pytest.mark.parametrize("delta", [1, 50, 700, 5000, 1 << 30])
def test_sssp_near_far_matches_dijkstra(coop, delta):
    for name in ["grid_w", "rmat_w", "disc_w", "path_w"]:
        g = SSSP_GRAPHS[name]()
        gd = _dev(g)
        s = gg.sample_sources(g, 1)[0]
        d, st = coop.sssp(gd, s, sssp_delta=delta)
        np.testing.assert_array_equal(_u32(d), tb.dijkstra(g, s))


def test_sssp_near_far_under_resizes(coop):
    g = SSSP_GRAPHS["grid_w"]()
    gd = _dev(g)
    ref = tb.dijkstra(g, 0)
    for seed in range(3):
        d, st = coop.sssp(gd, 0, sssp_delta=300, max_wgs=24, threads_per_wg=256, policy=coop.POLICY_RANDOM,
                          resize_prob=0.5, seed=seed, flags=coop.FLAG_CHECK, barriers_per_level=1 + seed % 2)
        np.testing.assert_array_equal(_u32(d), ref)


# ---------------------------------------------------------------- mid-interval offer_kill
@pytest.mark.parametrize("threads", [256, 1024])
def test_mid_interval_offer_kill_keeps_results_exact(coop, threads):
    """Demanded workgroups leave between the items of their static share (offer_kill
    inside the level) instead of waiting for the next resizing barrier,
    handing the rest of their share back; the survivors run it in a replay interval
    before the level ends.  Levels / distances stay bit-exact.  256 threads per workgroup run
    the scheduler-armed kernel specialisation, 1024 the general kernel's out-of-line instance."""
    info = coop.device_query(0, threads)
    N = info["max_coresident"] - 1
    g = gg.rmat(18, seed=3)
    gd = _dev(g)
    s = gg.sample_sources(g, 1)[0]
    ref = tb.bfs(g, s)
    mids = hbs = reps = 0
    for flags in (0, coop.FLAG_DIROPT):
        for q in (1, N // 2, N - 1):
            lv, st = coop.bfs(gd, s, flags=flags | coop.FLAG_CHECK, threads_per_wg=threads, policy=coop.POLICY_SCHEDULER,
                              task_wgs=q, task_blocks=N, task_block_ns=3_000, task_period_ns=15_000,
                              event_cap=1024)
            np.testing.assert_array_equal(lv.cpu().numpy(), ref)
            mids += st.mid_kills
            hbs += st.handbacks
            reps += st.replays
            assert st.handbacks <= st.mid_kills and (st.replays > 0) == (st.handbacks > 0)
    assert mids > 0
    if threads == 256:          # many CTAs with items left when asked: hand-backs and replays happen
        assert hbs > 0 and reps > 0
    gw = SSSP_GRAPHS["grid_w"]()
    d, st = coop.sssp(_dev(gw), 0, sssp_delta=500, threads_per_wg=threads, policy=coop.POLICY_SCHEDULER, task_wgs=N // 2,
                      task_blocks=N, task_block_ns=2_000, task_period_ns=10_000, flags=coop.FLAG_CHECK)
    np.testing.assert_array_equal(_u32(d), tb.dijkstra(gw, 0))


# ---------------------------------------------------------------- graph layout steps
def test_layout_kernels_match_numpy(coop):
    """coop_csr_probe / coop_csr_isolated / coop_csr_hub_first against their plain
    definitions on the host: probe = {degree | first neighbour}, isolated = degree-0
    bits, hub-first = each list a permutation of the original, by descending neighbour
    degree."""
    import ctypes
    lib = coop.load()
    for g in (gg.rmat(12, seed=5), gg.disjoint_union(gg.rmat(10, seed=3), gg.star(40)), gg.grid(9, 7)):
        gd = _dev(g)
        c, keep = coop._device_csr(gd, need_weights=False, probe=False)
        V, E = g.num_vertices, g.num_edges
        ro = g.row_offsets.numpy().astype(np.int64)
        col = g.col_idx.numpy().astype(np.int64)
        deg = np.diff(ro)
        probe = torch.empty(V, dtype=torch.int64, device="cuda")
        assert lib.coop_csr_probe(ctypes.byref(c), probe.data_ptr(), None) == 0
        p = probe.cpu().numpy().view(np.uint64)
        np.testing.assert_array_equal((p >> np.uint64(32)).astype(np.int64), deg)
        first = np.where(deg > 0, col[np.minimum(ro[:-1], max(E - 1, 0))], 0xFFFFFFFF)
        np.testing.assert_array_equal((p & np.uint64(0xFFFFFFFF)).astype(np.int64), first)
        iso = torch.empty((V + 31) // 32, dtype=torch.int32, device="cuda")
        assert lib.coop_csr_isolated(ctypes.byref(c), iso.data_ptr(), None) == 0
        bits = np.unpackbits(iso.cpu().numpy().view(np.uint8), bitorder="little")[:V]
        np.testing.assert_array_equal(bits.astype(bool), deg == 0)
        col2 = torch.empty(E, dtype=torch.int32, device="cuda")
        assert lib.coop_csr_hub_first(ctypes.byref(c), col2.data_ptr(), None) == 0
        h = col2.cpu().numpy().astype(np.int64)
        for v in range(V):
            a, b = ro[v], ro[v + 1]
            assert sorted(h[a:b]) == sorted(col[a:b])               # same neighbour set
            assert np.all(np.diff(deg[h[a:b]]) <= 0)                # descending neighbour degree
