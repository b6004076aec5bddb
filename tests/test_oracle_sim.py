"""Pins for O2/O3 (oracle/coop_sim.py, oracle/enumerate.py): the paper's
worked example (Fig. 1), the SPEC rule examples, closed forms, the textbook
oracle (itself pinned by scipy) and brute-force schedule enumeration."""
import itertools

import numpy as np
import pytest

import graphgen as gg
from conftest import golden
from oracle import coop_sim as cs
from oracle import enumerate as en
from oracle import textbook as tb


# ---------------- rules on the workgroup tuple ----------------
def test_fig1_worked_example():
    fx = golden("fig1_worked_example.json")
    N, M = fx["N"], fx["M_initial"]
    slots = [f"w{i}" for i in range(N)]
    for wg in fx["kill_order"]:
        M, killed = cs.rule_offer_kill(slots, M, wg, accept=True)
        assert killed
    assert M == fx["M_after_kills"] and slots[M:] == [None] * (N - M)
    M = cs.rule_request_fork(slots, M, N, fx["forking_workgroup"], len(fx["forked_ids"]), lambda i: f"new{i}")
    assert M == fx["M_after_fork"]
    assert [slots[i] for i in fx["forked_ids"]] == [f"new{i}" for i in fx["forked_ids"]]
    # killing in the other order is impossible: WG 2 is not the largest id while WG 3 lives
    slots = [f"w{i}" for i in range(N)]
    M, killed = cs.rule_offer_kill(slots, 4, 2, accept=True)
    assert not killed and M == 4


def test_spec_rule_examples():
    fx = golden("spec_rule_examples.json")
    for ex in fx["offer_kill"]:
        slots = [object() for _ in range(ex["M"])] + [None] * (ex["N"] - ex["M"])
        M, killed = cs.rule_offer_kill(slots, ex["M"], ex["wg"], ex["accept"])
        assert (M, killed) == (ex["M_after"], ex["killed"]), ex
        assert all(s is not None for s in slots[:M]) and all(s is None for s in slots[M:])
    for ex in fx["request_fork"]:
        slots = [("old", i) for i in range(ex["M"])] + [None] * (ex["N"] - ex["M"])
        if "error" in ex:
            with pytest.raises(cs.ForkBoundExceeded):
                cs.rule_request_fork(slots, ex["M"], ex["N"], ex["wg"], ex["k"], lambda i: ("new", i))
            continue
        M = cs.rule_request_fork(slots, ex["M"], ex["N"], ex["wg"], ex["k"], lambda i: ("new", i))
        assert M == ex["M_after"]
        assert [i for i in range(M) if slots[i][0] == "new"] == ex["new_ids"]


def test_fork_transmits_thread0_state_only():
    """S:76 / P:578-581: new threads hold exactly the transmit vars of thread 0."""
    g = gg.grid(4, 4)
    r = cs.simulate(g, 0, N=4, d=3, M0=1, scheduler=cs.SequenceScheduler([4]), chooser=cs.RandomChooser(1))
    assert r.episodes[0].forks == 3
    for tr in r.episodes[0].fork_transmit:
        assert set(tr) == set(cs.TRANSMIT)
        assert tr == r.episodes[0].wg0_transmit
    # at the first resizing barrier (after the swap of level 0) WG0 holds level 0, in=n1, out=n0
    assert r.episodes[0].wg0_transmit == {"level": 0, "in_sel": 1, "out_sel": 0}


# ---------------- config 1 ----------------
def test_c1_trace_and_levels():
    fx = golden("c1_trace.json")
    g = gg.grid(8, 8)
    for seed in range(20):
        r = cs.simulate(g, 0, N=fx["N"], d=fx["d"], M0=fx["M0"],
                        scheduler=cs.ScriptedScheduler({int(k): v for k, v in fx["script"].items()}, fx["M0"]),
                        chooser=cs.RandomChooser(seed))
        rr, cc = np.divmod(np.arange(64), 8)
        np.testing.assert_array_equal(r.values, rr + cc)                     # closed form
        assert r.m_trace == fx["m_after_episode"]
        assert (r.kills, r.forks) == (fx["kills"], fx["forks"])
        assert r.frontier_sizes == fx["level_sizes"]
        assert len(r.episodes) == 2 * len(fx["level_sizes"])


def test_c1_any_interleaving_any_order():
    """Fully random interleaving (primitives fire in any order): M' may fall short
    of the script's target, but levels never change."""
    g = gg.grid(8, 8)
    ref = tb.bfs(g, 0)
    for seed in range(30):
        r = cs.simulate(g, 0, N=4, d=4, scheduler=cs.RandomScheduler(seed, 0.4),
                        chooser=cs.RandomChooser(seed, prims_last=False))
        np.testing.assert_array_equal(r.values, ref)


# ---------------- random schedules vs textbook ----------------
@pytest.mark.parametrize("mk", [lambda: gg.rmat(7, seed=4), lambda: gg.binary_tree(5),
                                lambda: gg.disjoint_union(gg.path(6), gg.star(5)), lambda: gg.grid(3, 11)])
def test_bfs_random_schedules_match_textbook(mk):
    g = mk()
    for seed in range(8):
        s = gg.sample_sources(g, 8)[seed % 8] if g.num_edges else 0
        r = cs.simulate(g, s, N=5, d=2, M0=1 + seed % 5, scheduler=cs.RandomScheduler(seed, 0.5),
                        chooser=cs.RandomChooser(100 + seed, prims_last=seed % 2 == 0))
        np.testing.assert_array_equal(r.values, tb.bfs(g, s))
        assert r.frontier_sizes == tb.level_sizes(tb.bfs(g, s))


@pytest.mark.parametrize("mk", [lambda: gg.with_weights(gg.grid(7, 9), seed=2),
                                lambda: gg.with_weights(gg.rmat(7, seed=8), seed=3),
                                lambda: gg.with_constant_weights(gg.grid(5, 5), 3)])
def test_sssp_random_schedules_match_dijkstra(mk):
    g = mk()
    ref = tb.dijkstra(g, 0)
    for seed in range(6):
        r = cs.simulate(g, 0, mode="sssp", N=4, d=2, scheduler=cs.RandomScheduler(seed, 0.5),
                        chooser=cs.RandomChooser(seed, prims_last=seed % 2 == 1))
        np.testing.assert_array_equal(np.array(r.values, dtype=np.uint32), ref)


def test_sim_never_resize_and_empty_frontier():
    g = gg.empty(3)
    r = cs.simulate(g, 1, N=2, d=2)
    assert r.values == [-1, 0, -1] and len(r.episodes) == 2 and r.frontier_sizes == [1]
    with pytest.raises(ValueError):
        cs.simulate(g, 3, N=2, d=2)
    with pytest.raises(ValueError):
        cs.simulate(g, 0, N=2, d=2, M0=3)


# ---------------- O3: brute-force enumeration ----------------
def test_enumerate_all_resize_sequences_path4():
    g = gg.path(4)
    ref = tb.bfs(g, 0)
    n = 0
    seen_traces = set()
    for seq, r in en.all_resize_sequences(g, 0, N=3, d=1):
        np.testing.assert_array_equal(r.values, ref)
        assert len(r.episodes) == 8                      # 2 * (ecc + 1)
        seen_traces.add(tuple(r.m_trace))
        n += 1
    assert n == 3 ** 8
    assert len(seen_traces) == 3 ** 8                    # every schedule is realised


def test_enumerate_all_resize_sequences_grid3x3_sssp():
    g = gg.with_weights(gg.grid(3, 3), seed=4, wmax=5)
    ref = tb.dijkstra(g, 4)
    n = 0
    for seq, r in en.all_resize_sequences(g, 4, N=2, d=1, mode="sssp", episodes=None):
        np.testing.assert_array_equal(np.array(r.values, dtype=np.uint32), ref)
        n += 1
    assert n >= 2 ** 4


def test_enumerate_all_interleavings_tiny():
    """Every interleaving with at most 2 preemptions (CHESS-style bound) of
    2 WGs x 1 thread on a path-3 and a triangle, with a scripted kill+fork
    schedule: every run equals the textbook result."""
    for g, s in [(gg.path(3), 0), (gg.edges_to_csr(__import__("torch").tensor([0, 1, 2]),
                                                    __import__("torch").tensor([1, 2, 0]), 3), 1)]:
        ref = tb.bfs(g, s)
        runs = 0
        for r in en.all_interleavings(g, s, N=2, d=1,
                                      scheduler_factory=lambda: cs.SequenceScheduler([1, 2, 2, 1]),
                                      preemption_bound=2):
            np.testing.assert_array_equal(r.values, ref)
            runs += 1
        assert runs > 100


def test_enumeration_detects_a_broken_kernel(monkeypatch):
    """Non-vacuity: if forked workgroups received a wrong transmitted level, the
    enumeration would expose it."""
    g = gg.binary_tree(3)
    orig = cs.CoopSim._apply_fork

    def bad_fork(self, i):
        orig(self, i)
        for wg in self.slots[:self.M]:
            for t in wg:
                if t.env.get("level") is not None and t.wg != 0 and t.gb_passed == 0:
                    t.env["level"] += 1

    monkeypatch.setattr(cs.CoopSim, "_apply_fork", bad_fork)
    ref = tb.bfs(g, 0)
    bad = 0
    for seq, r in itertools.islice(en.all_resize_sequences(g, 0, N=2, d=1), 200):
        bad += not np.array_equal(r.values, ref)
    assert bad > 0


# ---------------- the paper's two barrier implementations and chunked intervals ----------------
VARIANTS = [(b, w) for b in ("desugared", "naive", "query") for w in ("stride", "chunk")] + [("query", "handback")]


@pytest.mark.parametrize("barrier,work", VARIANTS)
def test_barrier_variants_random_channel_bfs(barrier, work):
    """Naive and query resizing barriers, the chunk-counter
    distribution with offer_kill at chunk boundaries, and the GPU's static split
    with offer_kill between items and hand-back: levels equal O1 and the
    frontier sizes equal O1's per-level counts under random interleavings and resource
    messages posted at random times."""
    g = gg.rmat(8, seed=5)
    for s in gg.sample_sources(g, 2):
        ref = tb.bfs(g, s)
        for seed in range(6):
            d = 1 if work != "stride" else 2
            sch = cs.ChannelScheduler(seed=seed, rate=0.03, budget=8)
            r = cs.simulate(g, s, N=4, d=d, M0=4, scheduler=sch, barrier=barrier, work=work, chunk=2,
                            chooser=cs.RandomChooser(seed, prims_last=seed % 2 == 0))
            np.testing.assert_array_equal(r.values, ref)
            assert r.frontier_sizes == tb.level_sizes(ref)


@pytest.mark.parametrize("barrier,work", VARIANTS)
def test_barrier_variants_random_channel_sssp(barrier, work):
    g = gg.with_weights(gg.grid(6, 5), seed=2)
    ref = tb.dijkstra(g, 0)
    for seed in range(4):
        d = 1 if work != "stride" else 2
        sch = cs.ChannelScheduler(seed=seed, rate=0.03, budget=8)
        r = cs.simulate(g, 0, mode="sssp", N=4, d=d, M0=3, scheduler=sch, barrier=barrier, work=work,
                        chunk=3, chooser=cs.RandomChooser(seed))
        np.testing.assert_array_equal(np.array(r.values, dtype=np.uint64), ref.astype(np.uint64))


def test_naive_barrier_gathers_one_workgroup_per_call_in_ascending_arrival():
    """with the naive barrier, 'depending on order of arrival, it is possible that
    only one workgroup is killed per barrier call'.  Arrival in ascending id order: the slaves
    below the top offer while they are not the largest id (Kill-No-Op), so exactly one WG
    leaves per episode; arrival in descending order lets all of them go at once."""
    g = gg.path(12)
    asc = cs.simulate(g, 0, N=4, d=1, M0=4, scheduler=cs.ChannelScheduler(demand=3), barrier="naive",
                      chooser=cs.OrderedChooser(ascending=True))
    assert [e.kills for e in asc.episodes[:4]] == [1, 1, 1, 0]
    assert [e.M_after for e in asc.episodes[:3]] == [3, 2, 1]
    desc = cs.simulate(g, 0, N=4, d=1, M0=4, scheduler=cs.ChannelScheduler(demand=3), barrier="naive",
                       chooser=cs.OrderedChooser(ascending=False))
    assert desc.episodes[0].kills == 3 and desc.episodes[0].M_after == 1
    for r in (asc, desc):
        assert r.values == list(range(12)) and r.kills == 3


@pytest.mark.parametrize("ascending", [True, False])
def test_query_barrier_gathers_W_workgroups_in_one_call(ascending):
    """the master's query returns W = outstanding demand (capped at M-1, reading R5);
    ids >= M-W spin on offer_kill until claimed, so the whole demand is met at the first
    barrier whatever the arrival order."""
    g = gg.path(12)
    for D, expect in ((3, 3), (5, 3), (2, 2)):
        r = cs.simulate(g, 0, N=4, d=1, M0=4, scheduler=cs.ChannelScheduler(demand=D), barrier="query",
                        chooser=cs.OrderedChooser(ascending=ascending))
        assert r.episodes[0].query_W == expect and r.episodes[0].kills == expect
        assert r.episodes[0].M_after == 4 - expect
        assert r.values == list(range(12))


def test_chunked_interval_kill_between_chunks():
    """offer_kill at a chunk boundary takes a workgroup out in the middle of an
    interval, before any barrier; the chunk counter hands its remaining items to the others."""
    g = gg.grid(5, 5)
    r = cs.simulate(g, 0, N=4, d=1, M0=4, scheduler=cs.ChannelScheduler(demand=1), barrier="query",
                    work="chunk", chunk=1, chooser=cs.RandomChooser(3))
    assert r.mid_kills == 1 and r.kills == 1
    rr, cc = np.divmod(np.arange(25), 5)
    np.testing.assert_array_equal(r.values, rr + cc)


def test_handback_kill_between_items_replays_the_rest():
    """The GPU's mid-interval offer_kill: a demanded top workgroup leaves between the
    items of its static share and hands the rest back; the survivors run those items in a replay
    interval before the level ends (no fork, no query there).  Levels stay equal to O1, and
    hand-backs with items left (replay intervals) do happen under random interleavings."""
    g = gg.rmat(8, seed=5)
    s = gg.sample_sources(g, 1)[0]
    ref = tb.bfs(g, s)
    replays = mids = 0
    for seed in range(8):
        sch = cs.ChannelScheduler(posts={300 + 97 * seed: (2, 0), 3000 + 50 * seed: (0, 2)})
        r = cs.simulate(g, s, N=4, d=1, M0=4, scheduler=sch, barrier="query", work="handback",
                        chooser=cs.RandomChooser(seed))
        np.testing.assert_array_equal(r.values, ref)
        assert r.frontier_sizes == tb.level_sizes(ref)
        replays += r.replays
        mids += r.mid_kills
    assert mids > 0 and replays > 0


def test_naive_barrier_needs_the_published_group_count():
    """Reading R21: the naive barrier kills on entry, i.e. while slower workgroups may
    still be in the interval; if get_num_groups returned the live M, a slow workgroup could read a
    different value than its peers in the same interval (violating P:655-661, and its stride would
    skip or repeat items).  The simulator finds that interleaving; with the count published at the
    last release (what the GPU's per-CTA M is) every interleaving is exact (tests above)."""
    g = gg.rmat(8, seed=5)
    s = gg.sample_sources(g, 1)[0]
    hit = False
    for seed in range(30):
        try:
            cs.simulate(g, s, N=4, d=2, M0=4, scheduler=cs.ChannelScheduler(seed=seed, rate=0.05, budget=8),
                        barrier="naive", chooser=cs.RandomChooser(seed, prims_last=False), live_num_groups=True)
        except cs.SemanticsViolation as e:
            assert "get_num_groups changed" in str(e)
            hit = True
            break
    assert hit
