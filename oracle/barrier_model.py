"""O4: exhaustive model of the GPU resizing-barrier protocol (TEST INFRASTRUCTURE ONLY).

The CUDA runtimes (``csrc/coop_rt.cuh`` for the BFS/SSSP hot path,
``include/coop_device.cuh`` for user kernels) do not run the desugared
barrier/fork/barrier/kill/barrier form of the Resizing-Barrier rule
(PAPER.md:1573-1585); they collapse it into one episode on a packed word, in
the spirit of the paper's efficient "query" barrier, and
add kills outside the serial section (the naive barrier's arrival kill,
PAPER.md:918-934; offer_kill between the items of an interval with the rest of the
leaver's static share handed back to the survivors, and the device API's bare
offer_kill / request_fork).  The protocol is
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
  mid kill     (static items + hand-back) every member runs its static items
               (id, 0..K-1) of the level; after each item it reads demand d
               and W.M and stops when id + d >= W.M (id != 0); then loops:
               read W, read demand; resume if demand == 0 or id + demand < M
               or the generation moved; if id != M-1: resume for the rest of
               the interval (no more offers) once any CTA arrived, else spin;
               if id == M-1: CAS demand, hand back the items not yet run,
               kill-CAS W as above (on failure: withdraw them, return the
               demand unit, resume)
  replay       a serial section that finds handed-back items releases into a
               replay interval of the same level (no policy, M' = M, R flag):
               item i of the handed-back list runs on member i mod M
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
  P6 work coverage   -- with static items and hand-back, every item of a level
                        runs exactly once before the barrier that ends the level
                        releases (a leaver's unrun items run in replay intervals)

``bugs`` injects known-wrong protocol variants so the tests can show each
property is not vacuous; see :data:`BUGS`.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field, replace

# slot (pool) states per physical CTA
IDLE, CLAIMED, ASSIGNED, ACTIVE, TASK = "I", "C", "A", "X", "T"

# CTA program counters
(PARKED, IN_TASK, WAIT_GEN, WORK, HB_ITEM, HB_POLL, HB_POLLW, OFFER, OFFER_D, OFFER_CASD, DONATE,
 OFFER_CASW, WITHDRAW, REPLAY_RUN, ARRIVE, NV_D, NV_CASD, NV_CASW, SPIN, SER_POLICY, SER_CASD, SER_FORK,
 SER_RESET, SER_RELEASE, BK_R, BK_CASD, BK_CASW, BF_R, BF_CLAIM, BF_CASW, BF_ASSIGN, KILLED, EXITED) = range(33)

BUGS = {
    "kill_by_M_only": "a waiter decides its fate from R.M alone, ignoring that R may be a later generation",
    "no_wait_gen": "a forked CTA starts before the release of its generation",
    "midkill_wait_arrived": "mid-interval: a demanded non-top id keeps waiting for the top to leave even after "
                            "CTAs arrived (the rule before commit 2f99910)",
    "no_cap_on_behalf": "a leaver completing the episode forks up to N under a waiting policy although it is "
                        "not parked yet (ADVICE round 1, include/coop_device.cuh)",
    "handback_skips_item": "mid-interval: the leaver hands back from the item after the one in hand, "
                           "which it never finished",
    "kill_without_handback": "mid-interval: the leaver leaves without handing its unrun items back",
    "no_replay": "the serial section ignores handed-back items and ends the level",
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
    items: int = 0                  # 0: an interval's work is one step; K: K static items per member
                                    # with mid-interval offer_kill and hand-back (scheduler + query)
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
    released: bool = False
    mprime: int = -1                # M' published at the release
    level: int = 0                  # the level this interval belongs to (replay intervals repeat it)
    items: frozenset = frozenset()  # hand-back mode: the level's items (owner id, k)
    done: frozenset = frozenset()   #   items of the level run so far
    donated: frozenset = frozenset()  # items handed back in this interval (withdrawn ones removed)
    replay: tuple = ()              # a replay interval: the handed-back items it runs, in order


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
    return S((0, M0, 0), (0, M0, 0), 0, 0, (cfg.demand, cfg.withdraw, cfg.grant, cfg.bare), False, -1,
             slots, (None,) * P, ctas, (Gen(frozenset(range(M0)), frozenset(range(M0)), released=True, mprime=M0,
                                            items=_level_items(cfg, M0)),))


def _level_items(cfg: Cfg, M: int) -> frozenset:
    return frozenset((i, k) for i in range(M) for k in range(cfg.items))


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
                if s.hist[g].level >= E:    # forked at the final barrier
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
            if h.replay:
                nxt = Cta(REPLAY_RUN, c.lid, g)
            else:
                nxt = Cta(HB_ITEM, c.lid, g, (0, False)) if cfg.items else Cta(ARRIVE, c.lid, g)
            put(nxt, hist=hist, tpub=tpub)
            if cfg.bare and bl and not cfg.items:
                nb = (dl, wl, gl, bl - 1)
                if c.lid != 0:
                    put(Cta(BK_R, c.lid, g), hist=hist, tpub=tpub, budget=nb)
                put(Cta(BF_R, c.lid, g), hist=hist, tpub=tpub, budget=nb)
        # ---------------- static items, mid-interval offer_kill with hand-back ----------------
        elif c.pc == HB_ITEM:
            k, nostop = c.a
            h = s.hist[g]
            if k == cfg.items:
                put(Cta(ARRIVE, c.lid, g))
            else:
                it = (c.lid, k)
                if it in h.done:
                    raise ProtocolViolation(f"P6: item {it} of level {h.level} runs twice")
                put(Cta(HB_POLL, c.lid, g, (k + 1, nostop)), hist=_gh(s, g, done=h.done | {it}))
        elif c.pc == HB_POLL:                     # demand read with the item
            k, nostop = c.a
            midkill = sched and cfg.barrier == "query"
            if midkill and c.lid != 0 and not nostop and s.demand > 0:
                put(Cta(HB_POLLW, c.lid, g, (k, s.demand)))
            else:
                put(Cta(HB_ITEM, c.lid, g, (k, nostop)))
        elif c.pc == HB_POLLW:                    # ... and W.M: asked to surrender?
            k, d = c.a
            if c.lid + d >= s.W[1]:
                put(Cta(OFFER, c.lid, g, (k,)))
            else:
                put(Cta(HB_ITEM, c.lid, g, (k, False)))
        elif c.pc == OFFER:                       # loop head: read W
            put(Cta(OFFER_D, c.lid, g, (c.a[0], s.W)))
        elif c.pc == OFFER_D:                     # read demand, decide
            k, w = c.a
            d = s.demand
            wg, M, arr = w
            if d == 0 or c.lid == 0 or c.lid + d < M or wg != g:
                put(Cta(HB_ITEM, c.lid, g, (k, False)))
            elif c.lid != M - 1:
                if arr and "midkill_wait_arrived" not in bugs:
                    put(Cta(HB_ITEM, c.lid, g, (k, True)))      # no more offers this interval
                else:
                    put(Cta(OFFER, c.lid, g, (k,)))             # spin
            else:
                put(Cta(OFFER_CASD, c.lid, g, (k, w, d)))
        elif c.pc == OFFER_CASD:
            k, w, d = c.a
            if s.demand == d:
                put(Cta(DONATE, c.lid, g, (k, w)), demand=d - 1)
            else:
                put(Cta(OFFER, c.lid, g, (k,)))
        elif c.pc == DONATE:                      # hand back the items not yet run
            k, w = c.a
            k0 = k + 1 if "handback_skips_item" in bugs else k
            rem = frozenset((c.lid, j) for j in range(k0, cfg.items))
            if "kill_without_handback" in bugs:
                rem = frozenset()
            h = s.hist[g]
            put(Cta(OFFER_CASW, c.lid, g, (k, w, rem)), hist=_gh(s, g, donated=h.donated | rem))
        elif c.pc == OFFER_CASW:                  # kill_top: CAS W {g,M,a} -> {g,M-1,a}
            k, w, rem = c.a
            if s.W == w:
                out.extend(_kill_cas(s, p, c, w[1], w[2], cfg))
            elif s.W[0] != g or s.W[1] != c.lid + 1:
                put(Cta(WITHDRAW, c.lid, g, (k, rem)))           # M or gen moved: not the top now
            else:
                put(Cta(OFFER_CASW, c.lid, g, (k, s.W, rem)))    # arrivals raced the CAS
        elif c.pc == WITHDRAW:
            k, rem = c.a
            h = s.hist[g]
            put(Cta(HB_ITEM, c.lid, g, (k, False)), hist=_gh(s, g, donated=h.donated - rem), demand=s.demand + 1)
        elif c.pc == REPLAY_RUN:                  # this member's share of the handed-back items
            h = s.hist[g]
            M = h.mprime
            mine = [it for i, it in enumerate(h.replay) if i % M == c.lid]
            for it in mine:
                if it in h.done:
                    raise ProtocolViolation(f"P6: item {it} of level {h.level} runs twice")
            put(Cta(ARRIVE, c.lid, g), hist=_gh(s, g, done=h.done | frozenset(mine)))
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
            rg, rM, _ = s.R
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
            elif s.hist[rg].level >= E:
                put(Cta(EXITED), done=s.done or c.lid == 0, slots=_set(s.slots, p, IDLE))
            else:
                put(Cta(WORK, c.lid, rg))
        # ---------------- serial section ----------------
        elif c.pc == SER_POLICY:
            M, behalf = c.a
            wait = cfg.policy in ("scripted", "random")
            if cfg.items and s.hist[g].donated and "no_replay" not in bugs:
                put(Cta(SER_RESET, c.lid, g, (M, behalf, M, True)))     # a replay interval follows
                continue
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
                    put(Cta(SER_RESET, c.lid, g, (M, behalf, M + got, False)),
                        grant=s.grant - got if sf else s.grant)
                # else: wait for a CTA to park (self loop)
            else:
                put(Cta(SER_RESET, c.lid, g, (M, behalf, mp, False)), grant=s.grant - got if sf else s.grant)
        elif c.pc == SER_RESET:
            M, behalf, mp, rpl = c.a
            h = s.hist[g]
            if h.cur != h.arrived or h.todo:
                raise ProtocolViolation(f"P1: barrier {g} completes with arrivals {sorted(h.arrived)} "
                                        f"of members {sorted(h.cur)}")
            if rpl:
                ng = Gen(frozenset(range(mp)), frozenset(range(mp)), level=h.level, items=h.items, done=h.done,
                         replay=tuple(sorted(h.donated)))
            else:
                if cfg.items and h.done != h.items:
                    raise ProtocolViolation(f"P6: level {h.level} ends with items {sorted(h.items - h.done)} not run")
                ng = Gen(frozenset(range(mp)), frozenset(range(mp)), level=h.level + 1, items=_level_items(cfg, mp))
            put(Cta(SER_RELEASE, c.lid, g, (M, behalf, mp, rpl)), W=(g + 1, mp, 0), hist=s.hist + (ng,))
        elif c.pc == SER_RELEASE:
            M, behalf, mp, rpl = c.a
            hist = _set(s.hist, g + 1, replace(s.hist[g + 1], released=True, mprime=mp))
            st = replace(s, R=(g + 1, mp, int(rpl)), hist=hist)
            if behalf or c.lid >= mp:
                put(Cta(KILLED, c.lid, g), st)
            elif hist[g + 1].level >= E:
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
    max_level: int = 0
    replays: int = 0


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
    max_gen = max_level = replays = 0
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
        if s.W[0] < len(s.hist):
            max_level = max(max_level, s.hist[s.W[0]].level)
            if s.hist[s.W[0]].replay:
                replays += 1
        if not lst:
            if not all(c.pc == EXITED for c in s.ctas):
                raise ProtocolViolation(f"P5 deadlock: {_fmt(s)}")
            for g, h in enumerate(s.hist):
                if h.level < cfg.E and h.todo:
                    raise ProtocolViolation(f"P2: interval {g} ids {sorted(h.todo)} never worked")
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
    return Result(len(states), len(good), max_gen, max_level=max_level, replays=replays)


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
