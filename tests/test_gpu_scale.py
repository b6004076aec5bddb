"""GPU parity at (or near) the benchmarked configurations (VERDICT r1 "do this" 2):
the launch configuration bench.py times (512 threads/CTA, max co-resident CTAs,
direction-optimising BFS, full graph layout), SSSP on the 2048x2048 grid of
configs[1] against Dijkstra, the 64-bit row-offset path that single-GPU RMAT-27
needs, multitasked runs at RMAT-20, and compute-sanitizer runs of the
cooperative kernels.  Element-by-element comparison with the oracle."""
import os

import numpy as np
import pytest
import torch

import graphgen as gg
from oracle import textbook as tb

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def coop():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1707_01989_b200 import build, coop as c
    build.build()
    return c


@pytest.fixture(scope="module")
def rmat20():
    g = gg.rmat(20, seed=1, device="cuda")
    return g, g.to("cpu")


@pytest.mark.parametrize("diropt", [True, False])
def test_bfs_rmat20_bench_launch_config(coop, rmat20, diropt):
    """bench.py's launch: threads_per_wg=512, max_wgs=0 (max co-resident), FLAG_DIROPT,
    hub-first + probe + degree-zero layout; 6 sources."""
    g, gh = rmat20
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
    flags = coop.FLAG_DIROPT if diropt else 0
    for s in gg.sample_sources(gh, 6, seed=2):
        lv, st = coop.bfs(g, s, out, threads_per_wg=512, flags=flags)
        ref = tb.bfs(gh, s)
        np.testing.assert_array_equal(lv.cpu().numpy(), ref)
        assert st.reached == int((ref >= 0).sum())
        if diropt:
            assert st.bottom_up_levels >= 1


def test_bfs_rmat20_multitasked_query(coop, rmat20):
    """The multitasked configuration of the bench (scheduler CTA posting tasks every 200 us,
    Q = N/4, mid-interval offer_kill at chunk boundaries): levels exact for 4 sources."""
    g, gh = rmat20
    info = coop.device_query(0, 512)
    N = info["max_coresident"]
    q = max(1, (N - 1) // 4)
    for s in gg.sample_sources(gh, 4, seed=3):
        lv, st = coop.bfs(g, s, threads_per_wg=512, flags=coop.FLAG_DIROPT, policy=coop.POLICY_SCHEDULER,
                          task_wgs=q, task_blocks=4 * q, task_block_ns=20000, task_period_ns=30000,
                          task_first_ns=0, event_cap=1024)
        np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(gh, s))


@pytest.mark.parametrize("delta", [0, 64000])
def test_sssp_grid2048_configs1(coop, delta):
    """configs[1]: 2048x2048 grid, weights U[1,1000] per undirected pair (seed 1), from the
    corner and the centre; bench.py's two launch configurations (delta 0 / 64000)."""
    g = gg.with_weights(gg.grid(2048, 2048), seed=1)
    g.max_weight = 1000
    gd = g.to("cuda")
    gd.max_weight = 1000
    thr = 256 if delta == 0 else 512
    for s in (0, 1024 * 2048 + 1024):
        d, st = coop.sssp(gd, s, threads_per_wg=thr, max_wgs=148, sssp_delta=delta)
        np.testing.assert_array_equal(d.cpu().numpy().view(np.uint32), tb.dijkstra(g, s))
        assert st.episodes > 2000


@pytest.mark.parametrize("diropt", [True, False])
def test_bfs_forced_64bit_offsets(coop, diropt):
    """The uint64 row-offset instantiation (E >= 2^32, e.g. RMAT-27 on one GPU) forced on
    graphs the oracle finishes quickly, with and without the graph layout steps."""
    for g in (gg.rmat(16, seed=4), gg.disjoint_union(gg.rmat(12, seed=2), gg.grid(33, 17))):
        g64 = coop.with_offset_bits(g.to("cuda"), 64)
        flags = coop.FLAG_DIROPT if diropt else 0
        for s in gg.sample_sources(g, 3):
            lv, _ = coop.bfs(g64, s, flags=flags, threads_per_wg=512)
            np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(g, s))
            lv, _ = coop.bfs(g64, s, flags=flags, policy=coop.POLICY_RANDOM, resize_prob=0.5, seed=s,
                             threads_per_wg=256)
            np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(g, s))


def test_sssp_forced_64bit_offsets(coop):
    g = gg.with_weights(gg.rmat(14, seed=6), seed=3)
    g.max_weight = 1000
    g64 = coop.with_offset_bits(g.to("cuda"), 64)
    for s in gg.sample_sources(g, 2):
        d, _ = coop.sssp(g64, s, policy=coop.POLICY_RANDOM, resize_prob=0.3, seed=s)
        np.testing.assert_array_equal(d.cpu().numpy().view(np.uint32), tb.dijkstra(g, s))


@pytest.mark.parametrize("mode", ["standalone", "query", "naive"])
def test_bfs_source_loop_inside_one_launch(coop, mode):
    """coop_bfs_loop: BFS looped over sources inside one persistent launch, each
    restart a resizing barrier; under a periodic competing task (query / naive barrier) the
    scheduler kills and forks across runs.  The last run's levels are exact, every run
    completed, run end times increase."""
    g = gg.rmat(16, seed=3)
    gd = g.to("cuda")
    srcs = gg.sample_sources(g, 5, seed=4)
    kw = {}
    if mode != "standalone":
        kw = dict(policy=coop.POLICY_SCHEDULER, barrier_mode=coop.BARRIER_QUERY if mode == "query" else
                  coop.BARRIER_NAIVE, task_wgs=8, task_blocks=32, task_block_ns=20000, task_period_ns=200000,
                  task_first_ns=0, event_cap=4096)
    lv, runs, t_end, st = coop.bfs_loop(gd, srcs, 0.3, threads_per_wg=256, max_wgs=48, flags=coop.FLAG_DIROPT,
                                        **kw)
    assert runs > len(srcs)
    np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(g, srcs[(runs - 1) % len(srcs)]))
    assert np.all(np.diff(t_end) > 0) and t_end[-1] >= 0.3
    if mode != "standalone":
        assert st.kills > 0 and st.forks > 0 and st.tasks_completed > 0


def test_pipelined_async_bfs_calls(coop, rmat20):
    """bench.py's main-line form: asynchronous coop_bfs_launch calls, two in flight on one
    stream (workspaces 0/1), the control block initialised on the device and mirrored back by
    the kernel's last CTA; every output exact and the statistics belong to their own call."""
    g, gh = rmat20
    srcs = gg.sample_sources(gh, 6, seed=9)
    outs = [torch.empty(g.num_vertices, dtype=torch.int32, device="cuda") for _ in srcs]
    inflight, done = [], []
    for j, s in enumerate(srcs):
        inflight.append((j, coop.BfsCall(g, s, outs[j], threads_per_wg=512, flags=coop.FLAG_DIROPT, workspace=j % 2)))
        if len(inflight) == 2:
            j0, c0 = inflight.pop(0)
            done.append((j0, c0.wait()))
    for j0, c0 in inflight:
        done.append((j0, c0.wait()))
    deg = np.diff(gh.row_offsets.numpy())
    for j, st in done:
        ref = tb.bfs(gh, srcs[j])
        np.testing.assert_array_equal(outs[j].cpu().numpy(), ref)
        assert st.reached == int((ref >= 0).sum()) and st.kernel_ns > 0
