"""O4: exhaustive model of the GPU resizing-barrier protocol (TEST INFRASTRUCTURE ONLY).

The CUDA runtimes (``csrc/coop_rt.cuh`` for the BFS/SSSP hot path,
``include/coop_device.cuh`` for user kernels) do not run the desugared
barrier/fork/barrier/kill/barrier form of the Resizing-Barrier rule
(PAPER.md:1573-1585); they collapse it into one episode on a packed word, in
the spirit of the paper's efficient "query" barrier, and
add kills outside the serial section (the naive barrier's arrival kill,
PAPER.md:918-934; offer_kill at chunk boundaries inside an interval and the
device API's bare offer_kill / request_fork).  The protocol is
specified in DESIGN.md §4 and modelled here, independently of the CUDA source,
at the granularity of single atomic operations by thread 0 of each CTA:

  W = (gen, M, arrived)    arrival word (one 64-bit word)
  R = (gen, M)             release word (its own cache line)
  demand, grant            the scheduler channel

  arrive       old = atomicAdd(W.arrived, 1); last iff old.arrived+1 == old.M
  naive kill   (NAIVE barrier, id != 0) read W; while id == W.M-1 > 0 and
               demand > 0: CAS demand d -> d-1, then CAS W {g,M,a} -> {g,M-1,a}
               (retrying on concurrent arrivals); the leaver completes the
               episode on the waiters' behalf iff a == M-1
  mid kill     (chunk-counter intervals) a CTA whose claim saw
               id + demand >= W.M finishes its chunk, then loops: read W, read
               demand; give up if demand == 0 or id + demand < M or the
               generation moved; if id != M-1: resume claiming once any CTA
               arrived, else spin; if id == M-1: CAS demand, CAS W as above
  bare kill    (device API) id == W.M-1 > 0: take one demand unit (SCHEDULER)
               or accept (RANDOM), CAS W {g,M,a} -> {g,M-1,a} unless M or gen
               moved; completes the episode iff a == M-1
  bare fork    (device API) k from the grant (CAS) or RANDOM; claim up to k
               pool slots, CAS W {g,M,a} -> {g,M+got,a}, hand ids [M, M+got)
               to the claimed CTAs (mailbox; they join the current interval)
  serial       (last arriver or a leaver completing the episode; all others wait)
               M' from the policy -- SCRIPTED target / RANDOM any value /
               SCHEDULER query: take min(demand, M-1) by CAS, else fork
               min(grant, N-M); forks claim pool slots one at a time (SCRIPTED
               and RANDOM wait for enough parked CTAs, SCHEDULER takes what it
               finds); W := (gen+1, M', 0); R := (gen+1, M')
  waiters      spin until R.gen != gen; killed iff R.gen != gen+1 or id >= R.M
  park loop    on a mailbox: wait until R.gen == mailbox gen, then work;
               otherwise (optionally) leave the pool to run a task block

The scheduler's host side posts demand, withdraws it (task finished:
atomicExch(demand, 0)) and posts grants at nondeterministic times, within
per-run budgets.  Every reachable state under every interleaving is explored;
properties checked on every transition:

  P1 barrier safety  -- the barrier of interval g is released only when every
                        member of g arrived or left by a kill-CAS, and nobody
                        works in g+1 before that release
  P2 contiguity      -- the members of the current interval (start ids plus
                        forks minus kills) are exactly [0, W.M) after every
                        step; each works once
  P3 survivor prefix -- a waiter is killed iff its id >= M'
  P4 transmit        -- a CTA forked at a barrier gets WG 0's state published
                        at that barrier; a bare fork the forker's (P:572-584,
                        P:622-624)
  P5 liveness        -- from every reachable state some continuation ends with
                        every CTA exited (no deadlock, no livelock)
  P6 work coverage   -- with chunked intervals, every chunk of interval g is
                        processed before barrier g releases (a CTA leaves only
                        between chunks)

``bugs`` injects known-wrong protocol variants so the tests can show each
property is not vacuous; see :data:`BUGS`.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field, replace

# slot (pool) states per physical CTA
IDLE, CLAIMED, ASSIGNED, ACTIVE, TASK = "I", "C", "A", "X", "T"

# CTA program counters
(PARKED, IN_TASK, WAIT_GEN, WORK, CLAIM, PROC, OFFER, OFFER_D, OFFER_CASD, OFFER_CASW,
 ARRIVE, NV_D, NV_CASD, NV_CASW, SPIN, SER_POLICY, SER_CASD, SER_FORK, SER_RESET, SER_RELEASE,
 BK_R, BK_CASD, BK_CASW, BF_R, BF_CLAIM, BF_CASW, BF_ASSIGN, KILLED, EXITED) = range(29)

BUGS = {
    "kill_by_M_only": "a waiter decides its fate from R.M alone, ignoring that R may be a later generation",
    "no_wait_gen": "a forked CTA starts before the release of its generation",
    "midkill_wait_arrived": "mid-interval: a demanded non-top id keeps waiting for the top to leave even after "
                            "CTAs arrived (the rule before commit 2f99910)",
    "no_cap_on_behalf": "a leaver completing the episode forks up to N under a waiting policy although it is "
                        "not parked yet (ADVICE round 1, include/coop_device.cuh)",
    "kill_with_chunk": "mid-interval: a CTA offers itself before finishing the chunk in hand",
    "kill_any_top": "kill-CAS writes M-1 from a stale M after a concurrent fork moved W.M",
}


class ProtocolViolation(AssertionError):
    pass


@dataclass(frozen=True)
class Cfg:
    P: int                          # physical CTAs (N)
    M0: int
    E: int                          # intervals in the body (each ends with a resizing barrier)
    policy: str = "scripted"        # scripted | random | scheduler
    targets: tuple = ()             # scripted: M' per episode (0/absent = unchanged)
    barrier: str = "query"          # query | naive (scheduler policy)
    chunks: int = 0                 # 0: static split; C: chunk counter + mid-interval offer_kill
    bare: int = 0                   # device API: budget of bare offer_kill/request_fork calls per run
    demand: int = 0                 # host demand units (posted at nondeterministic times)
    withdraw: int = 0               # host withdrawals of outstanding demand
    grant: int = 0                  # host grant units
    tasks: bool = False             # parked CTAs may leave the pool for a task block
    bugs: frozenset = frozenset()


@dataclass(frozen=True)
class Cta:
    pc: int
    lid: int = -1
    gen: int = -1
    a: tuple = ()                   # pc-specific registers


@dataclass(frozen=True)
class Gen:
    cur: frozenset                  # current members: start ids + bare forks - kill-CAS leavers
    todo: frozenset                 # members that have not started their work of the interval
    arrived: frozenset = frozenset()
    claimed: int = 0                # chunk counter
    done: int = 0                   # chunks processed
    released: bool = False
    mprime: int = -1                # M' published at the release


@dataclass(frozen=True)
class S:
    W: tuple
    R: tuple
    demand: int
    grant: int
    budget: tuple                   # (demand, withdraw, grant, bare) left
    done: bool
    tpub: int                       # barrier at which WG 0 last published its transmit
    slots: tuple
    mail: tuple                     # per phys: (lid, gen, tx) or None
    ctas: tuple
    hist: tuple                     # per generation: Gen


def _initial(cfg: Cfg) -> S:
    P, M0 = cfg.P, cfg.M0
    ctas = tuple(Cta(WORK, p, 0) if p < M0 else Cta(PARKED) for p in range(P))
    slots = tuple(ACTIVE if p < M0 else IDLE for p in range(P))
    return S((0, M0, 0), (0, M0), 0, 0, (cfg.demand, cfg.withdraw, cfg.grant, cfg.bare), False, -1,
             slots, (None,) * P, ctas, (Gen(frozenset(range(M0)), frozenset(range(M0)), released=True, mprime=M0),))


def _set(t, i, v):
    return t[:i] + (v,) + t[i + 1:]


def _gh(s: S, g: int, **kw) -> tuple:
    return _set(s.hist, g, replace(s.hist[g], **kw))


def _check_members(s: S):
    g, M, _ = s.W
    if g < len(s.hist):
        if s.hist[g].cur != frozenset(range(M)):
            raise ProtocolViolation(f"P2: members of interval {g} are {sorted(s.hist[g].cur)}, W.M={M}")


def _successors(s: S, cfg: Cfg):
    out = []
    bugs = cfg.bugs
    P, E = cfg.P, cfg.E
    sched = cfg.policy == "scheduler"

    # ---------------- host side of the scheduler channel ----------------
    dl, wl, gl, bl = s.budget
    if not s.done:
        if dl:
            out.append(replace(s, demand=s.demand + 1, budget=(dl - 1, wl, gl, bl)))
        if wl and s.demand:
            out.append(replace(s, demand=0, budget=(dl, wl - 1, gl, bl)))
        if gl:
            out.append(replace(s, grant=s.grant + 1, budget=(dl, wl, gl - 1, bl)))

    for p, c in enumerate(s.ctas):
        def put(nc, st=None, **kw):
            base = st if st is not None else s
            out.append(replace(base, ctas=_set(base.ctas, p, nc), **kw))

        g = c.gen
        if c.pc == PARKED:
            if s.slots[p] == ASSIGNED:
                lid, mg, tx = s.mail[p]
                nxt = WORK if "no_wait_gen" in bugs else WAIT_GEN
                put(Cta(nxt, lid, mg), slots=_set(s.slots, p, ACTIVE))
            elif s.done and s.slots[p] == IDLE:
                put(Cta(EXITED), slots=_set(s.slots, p, IDLE))
            elif cfg.tasks and s.slots[p] == IDLE and not s.done:
                put(Cta(IN_TASK), slots=_set(s.slots, p, TASK))
        elif c.pc == IN_TASK:
            put(Cta(PARKED), slots=_set(s.slots, p, IDLE))
        elif c.pc == WAIT_GEN:
            if s.R[0] == g:
                if g >= E:                  # forked at the final barrier
                    put(Cta(EXITED), slots=_set(s.slots, p, IDLE))
                else:
                    put(Cta(WORK, c.lid, g))
            elif s.R[0] > g:
                raise ProtocolViolation("P1: forked CTA missed its generation")
        elif c.pc == WORK:
            if g >= len(s.hist) or not s.hist[g].released:
                raise ProtocolViolation(f"P1: work in interval {g} before its release")
            if g >= 1 and not s.hist[g - 1].released:
                raise ProtocolViolation(f"P1: work in interval {g} before barrier {g - 1} released")
            h = s.hist[g]
            if c.lid not in h.todo:
                raise ProtocolViolation(f"P2: id {c.lid} works in interval {g} (members {sorted(h.cur)}, "
                                        f"not started {sorted(h.todo)})")
            hist = _gh(s, g, todo=h.todo - {c.lid})
            tpub = g if c.lid == 0 else s.tpub          # WG 0 publishes its transmit state
            nxt = CLAIM if cfg.chunks else ARRIVE
            put(Cta(nxt, c.lid, g), hist=hist, tpub=tpub)
            if cfg.bare and bl and not cfg.chunks:
                nb = (dl, wl, gl, bl - 1)
                if c.lid != 0:
                    put(Cta(BK_R, c.lid, g), hist=hist, tpub=tpub, budget=nb)
                put(Cta(BF_R, c.lid, g), hist=hist, tpub=tpub, budget=nb)
        # ---------------- chunked interval ----------------
        elif c.pc == CLAIM:
            h = s.hist[g]
            ch = h.claimed
            midkill = sched and cfg.barrier == "query"
            stop = midkill and c.lid != 0 and s.demand > 0 and c.lid + s.demand >= s.W[1]
            hist = _gh(s, g, claimed=h.claimed + 1)
            if ch < cfg.chunks:
                if stop and "kill_with_chunk" in bugs:
                    put(Cta(OFFER, c.lid, g, (False,)), hist=hist)
                else:
                    put(Cta(PROC, c.lid, g, (stop,)), hist=hist)
            elif stop:
                put(Cta(OFFER, c.lid, g, (True,)), hist=hist)
            else:
                put(Cta(ARRIVE, c.lid, g), hist=hist)
        elif c.pc == PROC:
            h = s.hist[g]
            hist = _gh(s, g, done=h.done + 1)
            put(Cta(OFFER, c.lid, g, (False,)) if c.a[0] else Cta(CLAIM, c.lid, g), hist=hist)
        elif c.pc == OFFER:                       # loop head: read W
            put(Cta(OFFER_D, c.lid, g, (c.a[0], s.W)))
        elif c.pc == OFFER_D:                     # read demand, decide
            last_chunk, w = c.a
            d = s.demand
            wg, M, arr = w
            cont = Cta(ARRIVE, c.lid, g) if last_chunk else Cta(CLAIM, c.lid, g)
            if d == 0 or c.lid == 0 or c.lid + d < M or wg != g:
                put(cont)
            elif c.lid != M - 1:
                if arr and "midkill_wait_arrived" not in bugs:
                    put(cont)
                else:
                    put(Cta(OFFER, c.lid, g, (last_chunk,)))        # spin
            else:
                put(Cta(OFFER_CASD, c.lid, g, (last_chunk, w, d)))
        elif c.pc == OFFER_CASD:
            last_chunk, w, d = c.a
            if s.demand == d:
                put(Cta(OFFER_CASW, c.lid, g, (last_chunk, w, w[1])), demand=d - 1)
            else:
                put(Cta(OFFER, c.lid, g, (last_chunk,)))
        elif c.pc == OFFER_CASW:
            last_chunk, w, M = c.a
            if s.W == w:
                if w[1] != M and "kill_any_top" not in bugs:
                    raise ProtocolViolation(f"P2: kill-CAS writes M-1 from a stale M={M} (W.M={w[1]})")
                out.extend(_kill_cas(s, p, c, M, w[2], cfg))
            else:
                put(Cta(OFFER_CASW, c.lid, g, (last_chunk, s.W, M)))   # prev: keep M, new a
        # ---------------- arrival ----------------
        elif c.pc == ARRIVE:
            if sched and cfg.barrier == "naive" and c.lid != 0 and not c.a:
                put(Cta(NV_D, c.lid, g, (s.W,)))           # read W first
                continue
            wg, M, arr = s.W
            if wg != g:
                raise ProtocolViolation(f"P1: CTA {c.lid} arrives at barrier {g} but W is at {wg}")
            h = s.hist[g]
            hist = _gh(s, g, arrived=h.arrived | {c.lid})
            nW = (wg, M, arr + 1)
            if arr + 1 == M:
                put(Cta(SER_POLICY, c.lid, g, (M, False)), W=nW, hist=hist)
            else:
                put(Cta(SPIN, c.lid, g), W=nW, hist=hist)
        elif c.pc == NV_D:
            (w,) = c.a
            Mw = w[1]
            if c.lid != Mw - 1 or Mw <= 1 or s.demand == 0:
                put(Cta(ARRIVE, c.lid, g, ("add",)))
            else:
                put(Cta(NV_CASD, c.lid, g, (w, s.demand)))
        elif c.pc == NV_CASD:
            w, d = c.a
            if s.demand == d:
                put(Cta(NV_CASW, c.lid, g, (w,)), demand=d - 1)
            else:
                put(Cta(NV_D, c.lid, g, (w,)))             # `continue` keeps the old W snapshot
        elif c.pc == NV_CASW:
            (w,) = c.a
            if s.W == w:
                out.extend(_kill_cas(s, p, c, w[1], w[2], cfg))
            else:
                put(Cta(NV_CASW, c.lid, g, (s.W,)))        # prev: M and a re-read
        elif c.pc == SPIN:
            rg, rM = s.R
            if rg == g:
                continue
            if "kill_by_M_only" in bugs:
                killed = c.lid >= rM
            else:
                killed = rg != g + 1 or c.lid >= rM
            mp = s.hist[g + 1].mprime if g + 1 < len(s.hist) else None
            if mp is not None and killed != (c.lid >= mp) and "kill_by_M_only" not in bugs:
                raise ProtocolViolation(f"P3: id {c.lid} killed={killed} with M'={mp}")
            if killed:
                put(Cta(KILLED, c.lid, g))
            elif rg >= E:
                put(Cta(EXITED), done=s.done or c.lid == 0, slots=_set(s.slots, p, IDLE))
            else:
                put(Cta(WORK, c.lid, rg))
        # ---------------- serial section ----------------
        elif c.pc == SER_POLICY:
            M, behalf = c.a
            wait = cfg.policy in ("scripted", "random")
            if cfg.policy == "scripted":
                t = cfg.targets[g] if g < len(cfg.targets) else 0
                choices = [max(1, min(P, t)) if t else M]
            elif cfg.policy == "random":
                choices = list(range(1, P + 1))
            else:
                choices = None
            if choices is not None:
                for mp in choices:
                    if behalf and wait and "no_cap_on_behalf" not in bugs:
                        mp = min(mp, P - 1)
                    put(Cta(SER_FORK, c.lid, g, (M, behalf, mp, 0, wait, False)))
            elif cfg.barrier == "query" and s.demand and M > 1:
                put(Cta(SER_CASD, c.lid, g, (M, behalf, s.demand)))
            else:
                mp, sf = M, False
                if s.grant and M < P:
                    mp, sf = M + min(s.grant, P - M), True
                put(Cta(SER_FORK, c.lid, g, (M, behalf, mp, 0, False, sf)))
        elif c.pc == SER_CASD:
            M, behalf, d = c.a
            if s.demand == d:
                take = min(d, M - 1)
                put(Cta(SER_FORK, c.lid, g, (M, behalf, M - take, 0, False, False)), demand=d - take)
            else:
                put(Cta(SER_POLICY, c.lid, g, (M, behalf)))
        elif c.pc == SER_FORK:
            M, behalf, mp, got, wait, sf = c.a
            if M + got < mp:
                idle = [q for q in range(P) if s.slots[q] == IDLE]
                if idle:
                    if s.tpub != g:
                        raise ProtocolViolation(f"P4: fork at barrier {g} with WG 0's state of barrier {s.tpub}")
                    q = idle[0]             # claim the lowest pool bit
                    put(Cta(SER_FORK, c.lid, g, (M, behalf, mp, got + 1, wait, sf)),
                        slots=_set(s.slots, q, ASSIGNED), mail=_set(s.mail, q, (M + got, g + 1, ("wg0", g))))
                elif not wait:
                    put(Cta(SER_RESET, c.lid, g, (M, behalf, M + got)),
                        grant=s.grant - got if sf else s.grant)
                # else: wait for a CTA to park (self loop)
            else:
                put(Cta(SER_RESET, c.lid, g, (M, behalf, mp)), grant=s.grant - got if sf else s.grant)
        elif c.pc == SER_RESET:
            M, behalf, mp = c.a
            h = s.hist[g]
            if h.cur != h.arrived or h.todo:
                raise ProtocolViolation(f"P1: barrier {g} completes with arrivals {sorted(h.arrived)} "
                                        f"of members {sorted(h.cur)}")
            if cfg.chunks and h.done != cfg.chunks:
                raise ProtocolViolation(f"P6: barrier {g} completes with {h.done}/{cfg.chunks} chunks processed")
            hist = s.hist + (Gen(frozenset(range(mp)), frozenset(range(mp))),)
            put(Cta(SER_RELEASE, c.lid, g, (M, behalf, mp)), W=(g + 1, mp, 0), hist=hist)
        elif c.pc == SER_RELEASE:
            M, behalf, mp = c.a
            hist = _set(s.hist, g + 1, replace(s.hist[g + 1], released=True, mprime=mp))
            st = replace(s, R=(g + 1, mp), hist=hist)
            if behalf or c.lid >= mp:
                put(Cta(KILLED, c.lid, g), st)
            elif g + 1 >= E:
                put(Cta(EXITED), st, done=s.done or c.lid == 0, slots=_set(s.slots, p, IDLE))
            else:
                put(Cta(WORK, c.lid, g + 1), st)
        # ---------------- device API bare calls ----------------
        elif c.pc == BK_R:
            w = s.W
            accept = s.demand > 0 if sched else True    # RANDOM: the declining branch is WORK -> ARRIVE
            if accept and c.lid + 1 == w[1] and w[1] > 1:
                if sched:
                    put(Cta(BK_CASD, c.lid, g, (w, s.demand)))
                else:
                    put(Cta(BK_CASW, c.lid, g, (w, False)))
            else:
                put(Cta(ARRIVE, c.lid, g))
        elif c.pc == BK_CASD:
            w, d = c.a
            if s.demand == d:
                put(Cta(BK_CASW, c.lid, g, (w, True)), demand=d - 1)
            else:
                put(Cta(ARRIVE, c.lid, g))                 # declined (the CAS loop ended empty)
        elif c.pc == BK_CASW:
            w, took = c.a
            cur = s.W
            if "kill_any_top" not in bugs and (cur[1] != c.lid + 1 or cur[0] != g):
                put(Cta(ARRIVE, c.lid, g), demand=s.demand + (1 if took else 0))   # M moved: not killed
            elif cur == w:
                out.extend(_kill_cas(s, p, c, w[1], w[2], cfg))
            else:
                put(Cta(BK_CASW, c.lid, g, (cur, took)))
        elif c.pc == BF_R:
            M = s.W[1]
            if M < P:
                if sched:
                    if s.grant:
                        k = min(s.grant, P - M)
                        put(Cta(BF_CLAIM, c.lid, g, (k,)), grant=s.grant - k)
                    else:
                        put(Cta(ARRIVE, c.lid, g))
                else:
                    for k in range(1, P - M + 1):
                        put(Cta(BF_CLAIM, c.lid, g, (k,)))
                    put(Cta(ARRIVE, c.lid, g))
            else:
                put(Cta(ARRIVE, c.lid, g))
        elif c.pc == BF_CLAIM:
            (k,) = c.a
            idle = [q for q in range(P) if s.slots[q] == IDLE][:k]
            slots = s.slots
            for q in idle:
                slots = _set(slots, q, CLAIMED)
            back = (k - len(idle)) if sched else 0
            if idle:
                put(Cta(BF_CASW, c.lid, g, (tuple(idle), s.W)), slots=slots, grant=s.grant + back)
            else:
                put(Cta(ARRIVE, c.lid, g), grant=s.grant + back)
        elif c.pc == BF_CASW:
            phys, w = c.a
            if s.W == w:
                got = len(phys)
                base = w[1]
                h = s.hist[g]
                new = frozenset(range(base, base + got))
                hist = _gh(s, g, cur=h.cur | new, todo=h.todo | new)
                put(Cta(BF_ASSIGN, c.lid, g, (phys, base)), W=(w[0], base + got, w[2]), hist=hist)
            else:
                put(Cta(BF_CASW, c.lid, g, (phys, s.W)))
        elif c.pc == BF_ASSIGN:
            phys, base = c.a
            q = phys[0]
            slots = _set(s.slots, q, ASSIGNED)
            mail = _set(s.mail, q, (base, g, ("bare", c.lid, g)))
            rest = phys[1:]
            nc = Cta(BF_ASSIGN, c.lid, g, (rest, base + 1)) if rest else Cta(ARRIVE, c.lid, g)
            put(nc, slots=slots, mail=mail)
        elif c.pc == KILLED:
            put(Cta(PARKED), slots=_set(s.slots, p, IDLE))
    return out


def _kill_cas(s: S, p: int, c: Cta, M: int, a: int, cfg: Cfg):
    """Successful kill-CAS W {g, M, a} -> {g, M-1, a} by CTA p (id must be M-1)."""
    g = c.gen
    if c.lid != M - 1 or M <= 1:
        raise ProtocolViolation(f"P2: kill-CAS by id {c.lid} with M={M} (only id M-1 > 0 may leave, P:543-548)")
    h = s.hist[g]
    hist = _gh(s, g, cur=h.cur - {c.lid})
    nW = (g, M - 1, a)
    if a == M - 1:          # everybody else already waits: complete the episode on their behalf
        nc = Cta(SER_POLICY, c.lid, g, (M - 1, True))
    else:
        nc = Cta(KILLED, c.lid, g)
    return [replace(s, W=nW, hist=hist, ctas=_set(s.ctas, p, nc))]


@dataclass
class Result:
    states: int
    terminal: int
    max_gen: int = 0
    kills_seen: set = field(default_factory=set)


def explore_cfg(cfg: Cfg, max_states: int = 3_000_000) -> Result:
    """Explore every interleaving of ``cfg``; raise ProtocolViolation on any
    P1-P6 failure.  P5 is checked on the whole state graph: every reachable
    state must reach a state where all CTAs have exited."""
    for b in cfg.bugs:
        if b not in BUGS:
            raise ValueError(f"unknown bug {b}")
    init = _initial(cfg)
    ids = {init: 0}
    states = [init]
    succ: list[list[int]] = []
    q = deque([0])
    good = []
    max_gen = 0
    while q:
        i = q.popleft()
        s = states[i]
        nxt = _successors(s, cfg)
        lst = []
        for n in nxt:
            _check_members(n)
            j = ids.get(n)
            if j is None:
                j = len(states)
                ids[n] = j
                states.append(n)
                if j >= max_states:
                    raise RuntimeError("state budget exceeded")
                q.append(j)
            if j != i:
                lst.append(j)
        while len(succ) <= i:
            succ.append([])
        succ[i] = lst
        max_gen = max(max_gen, s.W[0])
        if not lst:
            if not all(c.pc == EXITED for c in s.ctas):
                raise ProtocolViolation(f"P5 deadlock: {_fmt(s)}")
            for g in range(cfg.E):
                if s.hist[g].todo:
                    raise ProtocolViolation(f"P2: interval {g} ids {sorted(s.hist[g].todo)} never worked")
            good.append(i)
    # P5 (liveness): backward reachability from the good terminal states
    pred: list[list[int]] = [[] for _ in states]
    for i, lst in enumerate(succ):
        for j in lst:
            pred[j].append(i)
    ok = bytearray(len(states))
    dq = deque(good)
    for i in good:
        ok[i] = 1
    while dq:
        j = dq.popleft()
        for i in pred[j]:
            if not ok[i]:
                ok[i] = 1
                dq.append(i)
    for i, flag in enumerate(ok):
        if not flag:
            raise ProtocolViolation(f"P5 livelock/deadlock: no continuation terminates from {_fmt(states[i])}")
    return Result(len(states), len(good), max_gen)


def _fmt(s: S) -> str:
    names = {v: k for k, v in globals().items() if isinstance(v, int) and k.isupper() and len(k) > 2
             and k not in ("IDLE",)}
    cs = ", ".join(f"{names.get(c.pc, c.pc)}(lid={c.lid},g={c.gen})" for c in s.ctas)
    return f"W={s.W} R={s.R} demand={s.demand} grant={s.grant} slots={''.join(s.slots)} [{cs}]"


def explore(P: int, M0: int, targets: list[int], episodes: int, max_states: int = 2_000_000,
            bugs=frozenset()):
    """Scripted-policy exploration (every interleaving, one target sequence):
    returns (n_states, n_terminal)."""
    r = explore_cfg(Cfg(P, M0, episodes, "scripted", tuple(targets), bugs=frozenset(bugs)), max_states)
    return r.states, r.terminal
