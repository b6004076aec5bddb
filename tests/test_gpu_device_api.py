"""GPU parity of the device API (include/coop_device.cuh): kernels written on
offer_kill / request_fork / global_barrier / resizing_global_barrier, through
the C ABI, against the oracle.

* Fig. 4 literally (coop_fig4_bfs) vs O1 textbook BFS, and the C1 scripted
  kill/fork trace vs O2 (the semantics simulator) and the golden trace.
* Cooperative work stealing (coop_work_steal, Fig. 2 + §3.2) vs O6: task count,
  per-depth histogram and the 64-bit value sum are schedule independent, so
  they must be bit-exact under any random or host-driven kill/fork schedule.
"""
import threading
import time

import numpy as np
import pytest
import torch

import graphgen as gg
from conftest import golden
from oracle import coop_sim as cs
from oracle import textbook as tb
from oracle import worksteal as ows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def coop():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1707_01989_b200 import build, coop as c
    build.build()
    return c


GRAPHS = {
    "grid8": lambda: gg.grid(8, 8),
    "grid_ragged": lambda: gg.grid(37, 53),
    "path300": lambda: gg.path(300),
    "star3000": lambda: gg.star(3000),
    "disconnected": lambda: gg.disjoint_union(gg.rmat(10, seed=3), gg.grid(9, 9)),
    "rmat12": lambda: gg.rmat(12, seed=1),
}


@pytest.mark.parametrize("name", list(GRAPHS))
def test_fig4_bfs_never_resize(coop, name):
    g = GRAPHS[name]()
    gd = g.to("cuda")
    with coop.DevHandle(policy=coop.POLICY_NEVER) as h:
        for s in [0] + gg.sample_sources(g, 2):
            lv, st = coop.fig4_bfs(h, gd, s)
            np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(g, s))
            ecc = int(tb.bfs(g, s).max())
            assert st["episodes"] == 2 * (ecc + 1)          # two resizing barriers per level
            assert st["kills"] == st["forks"] == 0


def test_fig4_c1_scripted_trace(coop):
    """Config 1 on the device API: 8x8 grid, N = 4, Fig. 4's two resizing
    barriers per level, the fixed schedule -> levels and the M trace equal O2's."""
    fx = golden("c1_trace.json")
    g = gg.grid(8, 8)
    script = [0] * 64
    for k, v in fx["script"].items():
        script[int(k)] = v
    sim = cs.simulate(g, 0, N=4, d=4, scheduler=cs.ScriptedScheduler({int(k): v for k, v in fx["script"].items()}, 4),
                      chooser=cs.RandomChooser(0))
    for threads in (128, 256, 512):
        with coop.DevHandle(max_wgs=4, policy=coop.POLICY_SCRIPTED, script=script, flags=coop.FLAG_CHECK,
                            m_trace_cap=64) as h:
            lv, st = coop.fig4_bfs(h, g.to("cuda"), 0, threads_per_wg=threads)
        np.testing.assert_array_equal(lv.cpu().numpy(), sim.values)
        assert st["m_trace"] == sim.m_trace == fx["m_after_episode"]
        assert (st["kills"], st["forks"]) == (fx["kills"], fx["forks"])
        assert st["episodes"] == 30 and st["violations"] == 0


@pytest.mark.parametrize("name", ["grid_ragged", "rmat12", "disconnected", "path300"])
def test_fig4_random_resizes(coop, name):
    g = GRAPHS[name]()
    gd = g.to("cuda")
    s = gg.sample_sources(g, 1)[0]
    ref = tb.bfs(g, s)
    for seed in range(3):
        with coop.DevHandle(max_wgs=48, init_wgs=1 + 9 * seed, policy=coop.POLICY_RANDOM, resize_prob=0.6,
                            seed=seed, flags=coop.FLAG_CHECK, m_trace_cap=4096) as h:
            lv, st = coop.fig4_bfs(h, gd, s)
        np.testing.assert_array_equal(lv.cpu().numpy(), ref)
        assert st["kills"] + st["forks"] > 0
        assert all(1 <= m <= 48 for m in st["m_trace"])


def test_fig4_host_scheduler_messages(coop):
    """Resource messages posted from another host thread while the kernel runs
    (query barrier): results stay exact and M moves."""
    g = gg.path(4000)                       # 4000 levels: the kernel runs for a while
    gd = g.to("cuda")
    with coop.DevHandle(max_wgs=32, policy=coop.POLICY_SCHEDULER, m_trace_cap=1 << 14) as h:
        def poster():
            for _ in range(5):
                time.sleep(0.002)
                h.demand(10)
                time.sleep(0.002)
                h.grant(8)
        th = threading.Thread(target=poster)
        th.start()
        lv, st = coop.fig4_bfs(h, gd, 0)
        th.join()
    np.testing.assert_array_equal(lv.cpu().numpy(), np.arange(4000, dtype=np.int32))
    assert all(1 <= m <= 32 for m in st["m_trace"])


TREES = [dict(seed=3, depth=12, max_fanout=4, rounds=2),
         dict(seed=2, depth=10, max_fanout=4, rounds=0),
         dict(seed=11, depth=6, max_fanout=3, fixed=True, rounds=1),
         dict(seed=5, depth=0, max_fanout=4, rounds=3)]


def _oracle(tr):
    return ows.run_stack(tr["seed"], tr["depth"], tr["max_fanout"], tr.get("fixed", False), tr["rounds"])


@pytest.mark.parametrize("ti", range(len(TREES)))
def test_work_steal_never(coop, ti):
    tr = TREES[ti]
    ref = _oracle(tr)
    for threads in (128, 256):
        with coop.DevHandle(policy=coop.POLICY_NEVER) as h:
            r, st = coop.work_steal(h, threads_per_wg=threads, **tr)
        assert (r["count"], r["total"], r["hist"]) == (ref["count"], ref["total"], ref["hist"])


@pytest.mark.parametrize("ti", range(3))
def test_work_steal_random_kill_fork(coop, ti):
    """Bare offer_kill / request_fork at the head of every loop iteration
    (§3.2): a workgroup may be killed with a non-empty queue (its tasks are
    stolen), forked workgroups read their own queue id after the fork point."""
    tr = TREES[ti]
    ref = _oracle(tr)
    kills = forks = 0
    for seed in range(4):
        with coop.DevHandle(max_wgs=64, init_wgs=8 + 16 * seed, policy=coop.POLICY_RANDOM, kill_prob=0.05,
                            fork_prob=0.02, max_fork=4, seed=seed, flags=coop.FLAG_CHECK) as h:
            r, st = coop.work_steal(h, **tr)
        assert (r["count"], r["total"], r["hist"]) == (ref["count"], ref["total"], ref["hist"])
        assert 1 <= st["min_m"] <= st["max_m"] <= 64
        kills += st["kills"]
        forks += st["forks"]
    if ref["count"] > 1000:
        assert kills > 0 and forks > 0


def test_work_steal_host_messages(coop):
    tr = dict(seed=3, depth=13, max_fanout=4, rounds=8)
    ref = _oracle(tr)
    with coop.DevHandle(max_wgs=96, policy=coop.POLICY_SCHEDULER) as h:
        def poster():
            for _ in range(4):
                time.sleep(0.001)
                h.demand(40)
                time.sleep(0.001)
                h.grant(30)
        th = threading.Thread(target=poster)
        th.start()
        r, st = coop.work_steal(h, **tr)
        th.join()
    assert (r["count"], r["total"], r["hist"]) == (ref["count"], ref["total"], ref["hist"])


def test_work_steal_queue_overflow_reported(coop):
    """A tree wider than the queues: the kernel aborts cleanly with COOP_ERR_OVERFLOW."""
    with coop.DevHandle(max_wgs=1) as h:
        with pytest.raises(coop.CoopError) as ei:
            coop.work_steal(h, seed=1, depth=4, max_fanout=16, fixed=True, queue_cap=8)
    assert ei.value.status == 7


# ---------------- Table 1's Pannotia applications on the device API ----------------
@pytest.mark.parametrize("app", ["color", "mis", "psssp"])
@pytest.mark.parametrize("policy", ["never", "random"])
def test_pannotia_apps_match_oracle(coop, app, policy):
    """color / mis / p-sssp as cooperative kernels with Table 1's resizing barriers,
    exact against oracle/pannotia.py (itself pinned by the greedy MIS, proper colouring,
    closed forms and Dijkstra), also under random kills and forks at every resizing barrier."""
    from oracle import pannotia as pn
    graphs = [gg.rmat(11, seed=3), gg.disjoint_union(gg.grid(23, 17), gg.star(300))]
    kw = dict(policy=coop.POLICY_NEVER) if policy == "never" else dict(
        max_wgs=24, init_wgs=5, policy=coop.POLICY_RANDOM, resize_prob=0.5, seed=7, flags=coop.FLAG_CHECK)
    for g in graphs:
        if app == "psssp":
            g = gg.with_weights(g, seed=4)
            g.max_weight = 1000
        gd = g.to("cuda")
        if app == "psssp":
            gd.max_weight = 1000
        ro, col = g.row_offsets.tolist(), g.col_idx.tolist()
        for arg in ([3, 11] if app != "psssp" else gg.sample_sources(g, 2)):
            with coop.DevHandle(**kw) as h:
                out, iters, st = coop.pannotia(h, app, gd, arg)
            got = out.cpu().numpy()
            if app == "color":
                ref, it = pn.color(ro, col, g.num_vertices, arg)
            elif app == "mis":
                ref, it = pn.mis(ro, col, g.num_vertices, arg)
            else:
                ref, it = pn.p_sssp(ro, col, [int(x) for x in g.weights.tolist()], g.num_vertices, arg)
                got = got.view(np.uint32)
            np.testing.assert_array_equal(got, ref)
            assert iters == it
            if policy == "random":
                assert st["kills"] + st["forks"] > 0
