"""O2: cooperative-kernel semantics simulator (TEST INFRASTRUCTURE ONLY).

Follows the operational semantics of PAPER.md Appendix A step by step
(rules in Fig. 7) and runs the cooperative graph
traversal of Fig. 4 as BFS or as worklist SSSP.

Kernel state: ``(sigma, (w_0 .. w_{M-1}, bot^{N-M}))``.
``sigma`` is the shared state (graph, level/dist arrays, node arrays n0/n1,
SSSP dedupe array); each workgroup is a d-tuple of thread states ``(l, ss)``:
``l`` is the thread's private environment (a dict) and ``ss`` -- the remaining
statements -- is a Python generator.  Every ``yield`` of a thread generator is
one statement boundary, so advancing a generator by one ``next()`` is exactly
one Thread-Step.

The four primitives are NOT thread steps; a thread that
reaches one blocks on it and the engine applies the matching rule:

* Kill-No-Op / Kill when all d threads of a workgroup are
  at the same ``offer_kill``.  Kill only for workgroup M-1 and only when M > 1
  (prose P:543-548; the rule's premise "M > 0" at P:1524 is read as M > 1 --
  DESIGN.md reading R1).
* Fork when all d threads of a workgroup are at the same
  ``request_fork``; the scheduler picks k in [0, N-M]; each new thread's
  environment is the *transmit-annotated* part of thread 0's environment
  (the §3.1 normative form -- Appendix A transmits the whole
  state as a stated simplification).
* Barrier when every thread of every active workgroup is
  at a ``global_barrier``; ``sync`` is a sequentially-consistent flush here
  (memory is SC in the simulator; reading R9).
* Resizing-Barrier is desugared: workgroup 0 executes
  ``GB; request_fork; GB; GB`` and every other workgroup ``GB; GB; offer_kill;
  GB`` (the rule's ``l_{1,j}`` / ``forall i != 1`` read as workgroup 0 --
  reading R2, consistent with P:622-624).  Barriers are matched by barrier
  instance (episode, index) rather than by identical continuation (reading R3).

Fig. 4's ``process_node`` is unspecified in the paper; reading R8:
BFS claims a neighbour with atomicMin(level[w], level+1) and appends it iff the
old value was INF; SSSP relaxes with atomicMin(dist[v], dist[u]+w) and appends
iff the distance improved and ``atomicMax(qlev[v], round+1) < round+1``.
Non-atomic pre-check reads are separate thread steps so that the interleaver
can race them against the atomics.

After every transition the engine asserts the invariants of SURVEY §8(c) O2
step 5 (M bounds, contiguity, kill only at M-1, fork framing, transmit
completeness, barrier safety, M constant inside a resizing-barrier interval).
Any violation raises :class:`SemanticsViolation`.
"""
from __future__ import annotations

import random
from dataclasses import dataclass, field
from typing import Callable, Optional

INF = 0xFFFFFFFF

# tokens a thread can block on
GB = "global_barrier"
OFFER_KILL = "offer_kill"
REQUEST_FORK = "request_fork"

TRANSMIT = ("level", "in_sel", "out_sel")       # Fig. 4 lines P:712-714


class SemanticsViolation(AssertionError):
    pass


class Deadlock(RuntimeError):
    pass


class ForkBoundExceeded(SemanticsViolation):
    pass


# --------------------------------------------------------------------------
# The primitive rules on the workgroup tuple (w_0..w_{M-1}, bot^{N-M})
# --------------------------------------------------------------------------
def rule_offer_kill(slots: list, M: int, wg: int, accept: bool) -> tuple[int, bool]:
    """Rules Kill-No-Op / Kill (prose P:541-548).

    ``slots`` is mutated in place.  Returns (M', killed).  Only the workgroup
    with the largest id, M-1, can be killed, never when M = 1 (reading R1);
    otherwise -- or if the scheduler declines -- the offer is a no-op.
    """
    if accept and wg == M - 1 and M > 1:
        slots[wg] = None
        return M - 1, True
    return M, False


def rule_request_fork(slots: list, M: int, N: int, wg: int, k: int, make_wg) -> int:
    """Rule Fork (prose P:564-581).

    k in [0, N-M] new workgroups get ids M..M+k-1; ``make_wg(new_id)`` builds
    each from the transmit-annotated state of thread 0 of ``wg``.  Returns M+k.
    k = 0 is always valid and forced when M = N.
    """
    if not (0 <= wg < M):
        raise SemanticsViolation("request_fork by an inactive workgroup (reading R4: m < M)")
    if not (0 <= k <= N - M):
        raise ForkBoundExceeded(f"k={k} outside [0, N-M]=[0,{N - M}] (P:565)")
    for a in range(k):
        slots[M + a] = make_wg(M + a)
    return M + k


# --------------------------------------------------------------------------
# Scheduler: the nondeterministic choices of Kill/Fork
# --------------------------------------------------------------------------
class Scheduler:
    """Base: never resizes (P:1079-1080 'forcing the scheduler to never modify')."""

    def target(self, episode: int, M: int, N: int) -> int:
        return M

    def accept_kill(self, episode: int, M: int, N: int) -> bool:
        return M > self.target(episode, M, N)

    def fork_count(self, episode: int, M: int, N: int) -> int:
        return max(0, min(self.target(episode, M, N) - M, N - M))


class NeverResize(Scheduler):
    pass


class ScriptedScheduler(Scheduler):
    """``script[e] = M'`` -- the target active count chosen at episode e.

    Entries persist: the target set at episode e applies to later episodes until
    the next script entry (so 'unchanged' episodes keep the current target).
    """

    def __init__(self, script: dict[int, int], M0: int):
        self.script = dict(script)
        self.M0 = M0

    def target(self, episode, M, N):
        t = self.M0
        for e in sorted(self.script):
            if e <= episode:
                t = self.script[e]
        return max(1, min(N, t))


class SequenceScheduler(Scheduler):
    """Target M' for episode e = seq[e] (e beyond the sequence: unchanged)."""

    def __init__(self, seq: list[int]):
        self.seq = list(seq)
        self.cur = None

    def target(self, episode, M, N):
        if episode < len(self.seq):
            return max(1, min(N, self.seq[episode]))
        return M


class RandomScheduler(Scheduler):
    """At each episode, with probability p pick M' ~ U[1, N] (seeded), else keep M."""

    def __init__(self, seed: int, p: float = 0.5):
        self.rng = random.Random(seed)
        self.p = p
        self.cache: dict[int, Optional[int]] = {}

    def target(self, episode, M, N):
        if episode not in self.cache:
            self.cache[episode] = self.rng.randint(1, N) if self.rng.random() < self.p else None
        t = self.cache[episode]
        return M if t is None else t


class ChannelScheduler(Scheduler):
    """The scheduler of §4.2 driven by resource messages:
    ``demand`` workgroups wanted back, ``grant`` workgroups that may join.
    Kill is accepted while demand is outstanding (one unit per kill); a fork
    takes min(grant, N-M).  ``query`` returns the outstanding demand capped at
    M-1.  Messages arrive at nondeterministic times: ``posts`` maps
    an engine transition count to (demand, grant) added at that point, and with
    ``rate`` > 0 a seeded RNG adds one unit of demand (or, half as often, grant)
    before a transition with that probability, up to ``budget`` units."""

    def __init__(self, posts: Optional[dict] = None, seed: int = 0, rate: float = 0.0, budget: int = 0,
                 demand: int = 0, grant: int = 0):
        self.posts = dict(posts or {})
        self.rng = random.Random(seed)
        self.rate = rate
        self.budget = budget
        self.demand = demand
        self.grant = grant
        self.reserved = 0            # query barrier: W frozen at the release (reading R17)

    def tick(self, t: int):
        if t in self.posts:
            dd, gg = self.posts[t]
            self.demand += dd
            self.grant += gg
        if self.budget and self.rate and self.rng.random() < self.rate:
            self.budget -= 1
            if self.rng.random() < 2 / 3:
                self.demand += 1
            else:
                self.grant += 1

    def target(self, episode, M, N):
        return M

    def accept_kill(self, episode, M, N):
        if self.reserved:
            self.reserved -= 1
            return True
        if self.demand:
            self.demand -= 1
            return True
        return False

    def fork_count(self, episode, M, N):
        k = min(self.grant, N - M)
        self.grant -= k
        return k

    def query(self, M):
        return min(self.demand, M - 1)


# --------------------------------------------------------------------------
# Interleaver: which enabled transition fires next
# --------------------------------------------------------------------------
class Chooser:
    """Picks among enabled transitions.  ``options`` is a list of
    (kind, payload) tuples with kind in {'step','kill','fork','barrier'}."""

    def choose(self, options: list) -> int:
        raise NotImplementedError


class RandomChooser(Chooser):
    """Seeded random interleaving.  With ``prims_last`` (default) workgroup-level
    primitives fire only when no thread step is enabled, highest workgroup id
    first -- a legal interleaving that lets the scheduler realise its target M'
    (only w_{M-1} may be killed, so kills must be offered in descending order)."""

    def __init__(self, seed: int, prims_last: bool = True):
        self.rng = random.Random(seed)
        self.prims_last = prims_last

    def choose(self, options):
        if self.prims_last:
            steps = [i for i, o in enumerate(options) if o[0] == "step"]
            if steps:
                return self.rng.choice(steps)
            prims = [i for i, o in enumerate(options) if o[0] in ("kill", "fork")]
            if prims:
                return max(prims, key=lambda i: options[i][1])
            return 0
        return self.rng.randrange(len(options))


class OrderedChooser(Chooser):
    """Deterministic: an enabled workgroup primitive fires at once (highest id
    first, so the scheduler can take the top workgroup); otherwise the thread
    step of the lowest (``ascending``) or highest workgroup id; a barrier when
    nothing else is enabled.  Makes workgroups reach a barrier in id order (the
    arrival orders of P:931-934)."""

    def __init__(self, ascending: bool = True):
        self.sign = 1 if ascending else -1

    def choose(self, options):
        def key(i):
            kind, pl = options[i]
            if kind == "barrier":
                return (2, 0)
            if kind == "step":
                return (1, self.sign * pl.wg)
            return (0, -pl)
        return min(range(len(options)), key=key)


class ReplayChooser(Chooser):
    """Deterministic replay of a choice prefix, then choice 0; records the
    branching factor at each point (for exhaustive DFS enumeration, O3).

    Choice 0 is always "keep running the thread that ran last" when that
    thread is still enabled, so a non-zero choice there is a *preemption*
    (used for preemption-bounded enumeration)."""

    def __init__(self, prefix: list[int]):
        self.prefix = list(prefix)
        self.pos = 0
        self.last = None
        self.trace: list[tuple[int, int, bool]] = []   # (chosen, n_options, continuation_available)

    def choose(self, options):
        perm = list(range(len(options)))
        cont = False
        for j, o in enumerate(options):
            if o[0] == "step" and o[1] is self.last:
                perm = [j] + [i for i in range(len(options)) if i != j]
                cont = True
                break
        c = self.prefix[self.pos] if self.pos < len(self.prefix) else 0
        self.pos += 1
        self.trace.append((c, len(options), cont))
        pick = perm[c]
        if options[pick][0] == "step":
            self.last = options[pick][1]
        return pick


# --------------------------------------------------------------------------
# Kernel state
# --------------------------------------------------------------------------
@dataclass
class Thread:
    wg: int               # workgroup id (slot index)
    lid: int              # local id in [0, d)
    env: dict
    gen: object = None    # generator = remaining statements ss
    blocked: Optional[tuple] = None   # token it waits on, or None if ready
    done: bool = False
    gb_passed: int = 0    # number of global barriers passed (safety check)


@dataclass
class Shared:
    """sigma: graph (immutable kernel parameters) + mutable arrays."""
    V: int
    ro: list
    col: list
    w: Optional[list]
    val: list                    # level[] (BFS) or dist[] (SSSP), INF = 0xFFFFFFFF
    nodes: list                  # [n0, n1]: each {'items': list, 'size': int}
    qlev: Optional[list] = None  # SSSP dedupe


@dataclass
class EpisodeRecord:
    episode: int
    M_before: int
    M_after: int = -1
    kills: int = 0
    forks: int = 0
    fork_transmit: list = field(default_factory=list)   # transmit env of each forked WG
    query_W: int = 0                                    # query barrier: W broadcast at the release
    mid_kills: int = 0                                  # kills at chunk boundaries after this barrier
    wg0_transmit: Optional[dict] = None                 # thread 0 of WG 0 at its request_fork


@dataclass
class SimResult:
    values: list                 # level (BFS, -1 unreachable) / dist (SSSP, INF unreachable)
    frontier_sizes: list         # in_nodes.size at each loop head with size > 0
    episodes: list               # EpisodeRecord per resizing barrier
    steps: int
    kills: int
    forks: int
    mid_kills: int = 0           # kills at chunk boundaries / between items inside an interval
    replays: int = 0             # hand-back: replay intervals run by the survivors

    @property
    def m_trace(self) -> list[int]:
        return [e.M_after for e in self.episodes]


class CoopSim:
    """Engine applying the Appendix A rules to a Fig. 4 kernel."""

    def __init__(self, V, ro, col, source, *, weights=None, N=4, d=4, M0=None,
                 scheduler: Optional[Scheduler] = None, chooser: Optional[Chooser] = None,
                 mode: str = "bfs", max_steps: int = 10_000_000, barrier: str = "desugared",
                 work: str = "stride", chunk: int = 1, live_num_groups: bool = False):
        if not (0 <= source < V):
            raise ValueError("source out of range")
        if mode not in ("bfs", "sssp"):
            raise ValueError(mode)
        if mode == "sssp" and weights is None:
            raise ValueError("sssp needs weights")
        self.N, self.d = N, d
        self.M = N if M0 is None else M0
        if not (1 <= self.M <= N):
            raise ValueError("need 1 <= M0 <= N (P:513-514)")
        self.mode = mode
        if barrier not in ("desugared", "naive", "query"):
            raise ValueError(barrier)
        if work not in ("stride", "chunk", "handback"):
            raise ValueError(work)
        if work in ("chunk", "handback") and d != 1:
            raise ValueError("the chunk-counter and hand-back variants are modelled at workgroup granularity "
                             "(d=1): the GPU decides to stop and leave CTA-collectively")
        if work == "handback" and barrier != "query":
            raise ValueError("hand-back runs with the query barrier (the GPU's SCHEDULER + query path)")
        if (barrier in ("naive", "query") or work != "stride") and not isinstance(scheduler, ChannelScheduler):
            raise ValueError("naive/query barriers and mid-interval kills are driven by a ChannelScheduler")
        self.barrier = barrier
        self.gbs = 3 if barrier == "desugared" else 2     # global barriers per resizing barrier
        self.work = work
        self.chunk = chunk
        self.counter = [0, 0]                             # chunk counters of n0/n1
        self.handed: list = []                            # hand-back: items handed back in this interval
        self.replay_items: list = []                      # ... run by the survivors in a replay interval
        self.replays = 0
        self.spin_W = 0                                   # query barrier: W broadcast at the release
        self.M_committed = None                           # query barrier: M - W until the spinners left
        self.mid_kills = 0
        self.live_num_groups = live_num_groups
        self.M_pub = self.M if M0 is None else M0                 # M published at the last release
        self.sched = scheduler or NeverResize()
        self.chooser = chooser or RandomChooser(0)
        self.max_steps = max_steps
        val = [INF] * V
        val[source] = 0
        n0 = {"items": [source] + [None] * (V - 1), "size": 1}
        n1 = {"items": [None] * max(V, 1), "size": 0}
        if mode == "sssp":
            # worklist may hold a vertex at most once per round (dedupe), but the
            # SSSP queue capacity must allow V entries per round
            pass
        self.sigma = Shared(V, list(ro), list(col), None if weights is None else list(weights),
                            val, [n0, n1], [0] * V if mode == "sssp" else None)
        self.slots: list[Optional[list[Thread]]] = [None] * N
        self.gb_fired = 0
        self.episodes: list[EpisodeRecord] = []
        self.frontier_sizes: list[int] = []
        self.steps = 0
        self.kills = 0
        self.forks = 0
        self.interval_M: Optional[int] = None    # M observed by get_num_groups in this interval
        for i in range(self.M):
            self.slots[i] = [self._new_thread(i, j, {}, resume=None) for j in range(d)]

    # ---------------- thread program (Fig. 4) ----------------
    def _new_thread(self, wg, lid, env, resume):
        t = Thread(wg, lid, env)
        t.gen = self._fig4(t, resume)
        return t

    def get_num_groups(self):
        # Reading R21: with the naive / query implementations get_num_groups is the count
        # published at the last release (M' of the query barrier excludes the W workgroups
        # committed to leave), not the live M: a fast workgroup's entry kill at the next
        # naive barrier, or a spinner not yet claimed, would otherwise change the value a
        # slow workgroup reads in the same interval (P:655-661 requires it constant).
        # ``live_num_groups`` reads the live M instead, to show that hazard.
        if self.barrier == "desugared" or self.live_num_groups:
            M = self.M
        else:
            M = self.M_pub
        if self.interval_M is None:
            self.interval_M = M
        elif self.interval_M != M:
            raise SemanticsViolation("get_num_groups changed inside a resizing-barrier interval (P:659-661)")
        return M

    def _resizing_barrier(self, t: Thread, which: int):
        """Desugared Resizing-Barrier rule (reading R2: master = WG 0),
        or the paper's two implementations of it (§4.2):

        naive  -- slaves offer_kill once on entry, then wait; the master waits for
                  the (possibly shrunk) M, calls request_fork (new WGs join the
                  waiting slaves), then releases;
        query  -- the master waits for everybody, calls request_fork, then query
                  (W), releases broadcasting W; ids >= M-W spin on offer_kill
                  until the scheduler claims them."""
        if self.barrier == "naive":
            if t.wg != 0:
                yield (OFFER_KILL, which)
                yield (GB, 0)
            else:
                yield (GB, 0)
                yield (REQUEST_FORK, which)
            yield (GB, 1)
            return
        if self.barrier == "query":
            yield (GB, 0)
            if self.replay_items:
                # hand-back: items handed back in the interval make this episode the start of
                # a replay interval -- the level is not over: no fork, no query (M' = M)
                yield (GB, 1)
                return "replay"
            if t.wg == 0:
                yield (REQUEST_FORK, which)
                if t.lid == 0:
                    W = self.sched.query(self.M)
                    self.sched.demand -= W             # frozen for this episode (reading R17)
                    self.sched.reserved += W
                    self.spin_W = W
                    self.M_committed = self.M - W if W else None
                    self.episodes[-1].query_W = W
                yield "step"
            yield (GB, 1)
            yield from self._query_spin(t, which)
            return
        if t.wg == 0:
            yield (GB, 0)
            yield (REQUEST_FORK, which)
            yield (GB, 1)
            yield (GB, 2)
        else:
            yield (GB, 0)
            yield (GB, 1)
            yield (OFFER_KILL, which)
            yield (GB, 2)

    def _process_node(self, t: Thread, node: int):
        s = self.sigma
        env = t.env
        out = s.nodes[env["out_sel"]]
        if self.mode == "bfs":
            L = env["level"]
            for e in range(s.ro[node], s.ro[node + 1]):
                w = s.col[e]
                pre = s.val[w]                      # non-atomic pre-check
                yield "step"
                if pre == INF:
                    old = s.val[w]                  # atomicMin(level[w], L+1)
                    s.val[w] = min(old, L + 1)
                    if old == INF:                  # push iff previously unvisited
                        out["items"][out["size"]] = w
                        out["size"] += 1
                    yield "step"
        else:
            r = env["level"]                        # round counter (transmitted)
            du = s.val[node]                        # read current dist[u]
            yield "step"
            for e in range(s.ro[node], s.ro[node + 1]):
                v = s.col[e]
                nd = du + s.w[e]
                if nd >= INF:
                    raise OverflowError("distance not representable in u32")
                pre = s.val[v]
                yield "step"
                if nd < pre:
                    old = s.val[v]                  # atomicMin(dist[v], nd)
                    s.val[v] = min(old, nd)
                    if nd < old:
                        q = s.qlev[v]               # atomicMax(qlev[v], r+1)
                        s.qlev[v] = max(q, r + 1)
                        if q < r + 1:
                            out["items"][out["size"]] = v
                            out["size"] += 1
                    yield "step"

    def _query_spin(self, t: Thread, which):
        # spin until claimed.  A non-top spinner's offers are Kill-No-Ops that
        # change nothing (stuttering), so it stays blocked until it is the top id.
        while t.wg != 0 and self.M_committed is not None and t.wg >= self.M_committed:
            yield (OFFER_KILL, which, "spin")

    def _chunk_loop(self, t: Thread):
        """Chunk-counter distribution of one interval (d=1): the workgroup claims
        ``chunk`` items at a time from the in-queue's atomic counter, so work is
        never tied to (id, M) and a workgroup may offer_kill between chunks
         without stranding items -- the remedy for wide graphs whose
        resizing barriers are rare.  Query style: a
        workgroup with id >= M - demand stops after its chunk and offers until
        claimed; only the top id can go; once some workgroup waits at the barrier
        the rest resume claiming and leave the demand to the barrier."""
        s = self.sigma
        env = t.env
        while True:
            c = self.counter[env["in_sel"]]             # atomicAdd(counter, chunk)
            self.counter[env["in_sel"]] = c + self.chunk
            sched = self.sched
            stop = t.wg != 0 and sched.demand > 0 and t.wg + sched.demand >= self.M
            yield "step"
            size = s.nodes[env["in_sel"]]["size"]
            for i in range(c, min(c + self.chunk, size)):
                node = s.nodes[env["in_sel"]]["items"][i]
                yield "step"
                yield from self._process_node(t, node)
            while stop:
                sched = self.sched
                if sched.demand == 0 or t.wg + sched.demand < self.M:
                    break
                if t.wg == self.M - 1:
                    yield (OFFER_KILL, "mid")              # accepted: this generator is dropped
                    break
                if any(th.blocked is not None and th.blocked[0] == GB
                       for th in self._active()):
                    break                                 # someone arrived: resume claiming
                yield "step"                              # spin
            if c >= size:
                return False

    def _handback_loop(self, t: Thread):
        """The GPU's SCHEDULER + query distribution (d=1): Fig. 4's static
        stride over the in-queue; after each item a workgroup with id >=
        M - demand stops and offers itself (query style); only the top id
        can go, and it hands the items of its stride it has not run back
        first; once some workgroup waits at the barrier the others resume and stop
        offering for the rest of the interval.  A Kill-No-Op withdraws the hand-back."""
        s = self.sigma
        env = t.env
        M = self.get_num_groups()
        items = s.nodes[env["in_sel"]]["items"]
        size = s.nodes[env["in_sel"]]["size"]
        yield "step"
        i, nostop = t.wg, False
        while i < size:
            node = items[i]
            yield "step"
            yield from self._process_node(t, node)
            i += M
            sched = self.sched
            stop = not nostop and t.wg != 0 and sched.demand > 0 and t.wg + sched.demand >= self.M
            yield "step"
            while stop:
                sched = self.sched
                if sched.demand == 0 or t.wg + sched.demand < self.M:
                    break
                if t.wg == self.M - 1:
                    rem = [items[j] for j in range(i, size, M)]
                    self.handed.extend(rem)                # hand back, then offer
                    yield (OFFER_KILL, "mid")              # accepted: this generator is dropped
                    if rem:                                # Kill-No-Op: withdraw
                        del self.handed[-len(rem):]
                    break
                if any(th.blocked is not None and th.blocked[0] == GB for th in self._active()):
                    nostop = True                         # someone arrived: no more offers
                    break
                yield "step"                              # spin
        return False

    def _fig4(self, t: Thread, resume):
        s = self.sigma
        env = t.env
        if resume is None:
            # transmit int level = 0; transmit in_nodes = n0; transmit out_nodes = n1
            env["level"] = 0
            env["in_sel"] = 0
            env["out_sel"] = 1
            yield "step"
            state = "head"
        else:
            # forked inside resizing barrier `resume`: continuation after request_fork
            # is "global_barrier(); global_barrier(); ss"; in the naive/query
            # implementations new WGs join the waiting slaves
            yield (GB, 1)
            if self.barrier == "desugared":
                yield (GB, 2)
            elif self.barrier == "query":
                yield from self._query_spin(t, resume)   # new WGs are slaves too
            state = "after_rb1" if resume == 1 else "head"
        while True:
            if state == "after_rb1":
                s.nodes[env["out_sel"]]["size"] = 0        # reset(out_nodes)  (reading R9: idempotent)
                self.counter[env["in_sel"]] = 0            # chunk counter of the next in-queue (idem)
                yield "step"
                env["level"] += 1                            # level++
                yield "step"
                yield from self._resizing_barrier(t, 2)
                state = "head"
            # while (in_nodes.size > 0)
            size = s.nodes[env["in_sel"]]["size"]
            if t.wg == 0 and t.lid == 0:
                self.frontier_sizes.append(size) if size > 0 else None
            yield "step"
            if size == 0:
                return
            if self.work == "chunk":
                killed = yield from self._chunk_loop(t)
                if killed:
                    return
                env["in_sel"], env["out_sel"] = env["out_sel"], env["in_sel"]
                yield "step"
                yield from self._resizing_barrier(t, 1)
                state = "after_rb1"
                continue
            if self.work == "handback":
                yield from self._handback_loop(t)
                env["in_sel"], env["out_sel"] = env["out_sel"], env["in_sel"]
                yield "step"
                while (yield from self._resizing_barrier(t, 1)) == "replay":
                    # replay interval: handed-back item j runs on workgroup j mod M
                    env["in_sel"], env["out_sel"] = env["out_sel"], env["in_sel"]
                    M = self.get_num_groups()
                    for j in range(t.wg, len(self.replay_items), M):
                        yield "step"
                        yield from self._process_node(t, self.replay_items[j])
                    env["in_sel"], env["out_sel"] = env["out_sel"], env["in_sel"]
                    yield "step"
                state = "after_rb1"
                continue
            # re-chunk: tid = get_global_id(); stride = get_global_size()
            M = self.get_num_groups()
            tid = t.wg * self.d + t.lid
            stride = M * self.d
            yield "step"
            i = tid
            while i < s.nodes[env["in_sel"]]["size"]:
                node = s.nodes[env["in_sel"]]["items"][i]
                yield "step"
                yield from self._process_node(t, node)
                i += stride
            # swap(&in_nodes, &out_nodes)
            env["in_sel"], env["out_sel"] = env["out_sel"], env["in_sel"]
            yield "step"
            yield from self._resizing_barrier(t, 1)
            state = "after_rb1"

    # ---------------- engine ----------------
    def _active(self):
        return [t for wg in self.slots if wg is not None for t in wg if not t.done]

    def _check_invariants(self):
        M = self.M
        if not (1 <= M <= self.N):
            raise SemanticsViolation(f"M={M} outside [1,N] (S:109)")
        for i in range(self.N):
            if (self.slots[i] is not None) != (i < M):
                raise SemanticsViolation(f"slots not contiguous: slot {i}, M={M} (P:512-513)")
        if self.slots[0] is None:
            raise SemanticsViolation("workgroup 0 killed (P:543)")

    def _advance(self, t: Thread):
        self.steps += 1
        if self.steps > self.max_steps:
            raise RuntimeError("step budget exceeded")
        try:
            tok = next(t.gen)
        except StopIteration:
            t.done = True
            t.blocked = None
            return
        t.blocked = None if tok == "step" else tok

    def _enabled(self):
        opts = []
        active = self._active()
        for t in active:
            if t.blocked is None:
                opts.append(("step", t))
        # workgroup-level primitives: all d threads at the same primitive token
        for i in range(self.M):
            wg = self.slots[i]
            toks = {t.blocked for t in wg}
            if len(toks) == 1:
                tok = next(iter(toks))
                if tok is not None and tok[0] == OFFER_KILL:
                    if len(tok) < 3 or i == self.M - 1:
                        opts.append(("kill", i))
                elif tok is not None and tok[0] == REQUEST_FORK:
                    opts.append(("fork", i))
        # global barrier: every thread of every active WG at a GB
        if active and all(t.blocked is not None and t.blocked[0] == GB for t in active):
            if all(not t.done for wg in self.slots[:self.M] for t in wg):
                opts.append(("barrier", None))
        return opts

    def _episode(self):
        return self.gb_fired // self.gbs

    def _apply_barrier(self):
        active = self._active()
        toks = {t.blocked for t in active}
        if len(toks) != 1:
            raise SemanticsViolation(f"barrier divergence: {toks} (S:83)")
        idx = next(iter(toks))[1]
        if idx != self.gb_fired % self.gbs:
            raise SemanticsViolation("barrier instance mismatch (reading R3)")
        passed = {t.gb_passed for t in active}
        # forked threads join at GB index 1; they did not pass GB 0 of this episode
        e = self._episode()
        if idx == 0:
            self._record(e)
            self.interval_M = None
            if self.work == "handback":                   # the interval's hand-backs are final
                self.replay_items, self.handed = self.handed, []
                self.replays += 1 if self.replay_items else 0
        for t in active:
            t.blocked = None
            t.gb_passed += 1
        self.gb_fired += 1
        if idx == self.gbs - 1:
            rec = self.episodes[-1]
            rec.M_after = self.M if self.M_committed is None else self.M_committed
            self.M_pub = rec.M_after
            self.interval_M = None
        del passed

    def _record(self, e):
        if len(self.episodes) <= e:
            self.episodes.append(EpisodeRecord(e, self.M))
        return self.episodes[e]

    def _apply_kill(self, i):
        e = self._episode()
        M = self.M
        wg = self.slots[i]
        which = wg[0].blocked[1]
        accept = i == M - 1 and self.sched.accept_kill(e, M, self.N)
        self.M, killed = rule_offer_kill(self.slots, M, i, accept)
        if killed:
            self.kills += 1
            if which == "mid":
                self.mid_kills += 1
            elif self.barrier == "naive":                 # on entry, before the episode's barrier
                self._record(e).kills += 1
            else:                                         # inside the episode / query spinners after it
                self.episodes[-1].kills += 1
            if self.M_committed is not None and self.M == self.M_committed:
                self.M_committed = None                   # every spinner has left
        else:
            for t in wg:                           # Kill-No-Op: advance past offer_kill
                t.blocked = None

    def _apply_fork(self, i):
        e = self._episode()
        M, N = self.M, self.N
        k = self.sched.fork_count(e, M, N)
        wg = self.slots[i]
        t0 = wg[0]
        which = t0.blocked[1]
        snap = {v: t0.env[v] for v in TRANSMIT}     # thread 0's transmit vars
        if i == 0:
            self.episodes[-1].wg0_transmit = dict(snap)

        def make_wg(new_id):
            threads = [self._new_thread(new_id, j, dict(snap), resume=which) for j in range(self.d)]
            for t in threads:
                if set(t.env) != set(TRANSMIT):
                    raise SemanticsViolation("transmit completeness (S:113)")
            self.episodes[-1].fork_transmit.append(dict(snap))
            return threads

        self.M = rule_request_fork(self.slots, M, N, i, k, make_wg)
        self.forks += k
        self.episodes[-1].forks += k
        for t in wg:
            t.blocked = None

    def run(self) -> SimResult:
        self._check_invariants()
        while True:
            opts = self._enabled()
            if not opts:
                if all(t.done for t in self._active()) and not self._active():
                    break
                if any(not t.done for t in self._active()):
                    raise Deadlock("no enabled transition (S:289)")
                break
            if isinstance(self.sched, ChannelScheduler):
                self.sched.tick(self.steps + self.gb_fired)
                opts = self._enabled()
            c = self.chooser.choose(opts)
            kind, payload = opts[c]
            if kind == "step":
                self._advance(payload)
            elif kind == "kill":
                self._apply_kill(payload)
            elif kind == "fork":
                self._apply_fork(payload)
            else:
                self._apply_barrier()
            self._check_invariants()
        vals = list(self.sigma.val)
        if self.mode == "bfs":
            vals = [-1 if x == INF else x for x in vals]
        return SimResult(vals, self.frontier_sizes, self.episodes, self.steps, self.kills, self.forks,
                         self.mid_kills, self.replays)


def simulate(g, source, *, mode="bfs", N=4, d=4, M0=None, scheduler=None, chooser=None,
             max_steps=10_000_000, barrier="desugared", work="stride", chunk=1,
             live_num_groups=False) -> SimResult:
    """Convenience wrapper over a graphgen.CSR."""
    ro = g.row_offsets.cpu().tolist()
    col = g.col_idx.cpu().tolist()
    w = None if g.weights is None else [int(x) & 0xFFFFFFFF for x in g.weights.cpu().tolist()]
    return CoopSim(g.num_vertices, ro, col, source, weights=w, N=N, d=d, M0=M0,
                   scheduler=scheduler, chooser=chooser, mode=mode, max_steps=max_steps,
                   barrier=barrier, work=work, chunk=chunk, live_num_groups=live_num_groups).run()
