"""O4: exhaustive model of the GPU resizing-barrier protocol (TEST INFRASTRUCTURE ONLY).

The CUDA runtime does not run the desugared barrier/fork/barrier/kill/barrier
form of the Resizing-Barrier rule; it collapses it into
one episode on a packed word, in the spirit of the paper's efficient
"query" barrier.  The protocol is specified in DESIGN.md §4
and modelled here, independently of the CUDA source, at the granularity of
single atomic operations by thread 0 of each CTA:

  W = (gen, M, arrived)                 arrival word (one 64-bit word)
  R = (gen, M)                          release word (its own cache line)
  arrive:    old = atomicAdd(W.arrived, 1); last iff old.arrived + 1 == old.M
  serial:    (last arriver only; all M CTAs are waiting)
             M' = policy(gen); for each new id in [M, M'): CAS an IDLE slot
             to CLAIMED, write its mailbox {id, gen+1, M', transmit of WG 0},
             store ASSIGNED; then W := (gen+1, M', 0)         (reset arrivals)
             and R := (gen+1, M')                              (release)
  waiters:   spin until R.gen != gen; killed iff R.gen != gen+1 or id >= R.M
  killed:    slot := IDLE, back to the park loop
  park loop: on ASSIGNED read mailbox, slot := ACTIVE, wait until
             R.gen == mailbox.gen, then run the body after the barrier

Every reachable state under every interleaving (and every scripted target
sequence) is explored; properties checked on every transition:

  P1 barrier safety  -- no CTA works in interval g+1 before all M_g CTAs
                        arrived at barrier g
  P2 contiguity      -- the ids working in interval g are exactly [0, M_g),
                        each once
  P3 survivor prefix -- ids [0, min(M, M')) are never killed
  P4 transmit        -- a forked CTA's transmit equals WG 0's at that barrier
                        
  P5 no deadlock     -- every terminal state has every CTA exited
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass

IDLE, CLAIMED, ASSIGNED, ACTIVE = 0, 1, 2, 3

# CTA program counters
PARKED, WAIT_GEN, WORK, ARRIVE, SPIN, SERIAL, RELEASE, KILLED, EXITED, RELEASE_R = range(10)


class ProtocolViolation(AssertionError):
    pass


@dataclass(frozen=True)
class Cta:
    pc: int
    lid: int = -1
    gen: int = -1
    M: int = -1
    claim_next: int = 0       # serial section: next new id to place
    mprime: int = -1


def _initial(P, M0):
    ctas = tuple(Cta(WORK, p, 0, M0) if p < M0 else Cta(PARKED) for p in range(P))
    slots = tuple(ACTIVE if p < M0 else IDLE for p in range(P))
    mail = tuple((-1, -1, -1, -1) for _ in range(P))
    W = ((0, M0, 0), (0, M0))      # (arrival word, release word)
    worked = ((),)            # per gen: tuple of lids that worked
    arrivals = (0,)           # per gen: arrivals
    m_at = (M0,)              # per gen: M of that interval
    return (W, slots, mail, -1, False, ctas, worked, arrivals, m_at)


def _successors(state, targets, P, E, bugs=frozenset()):
    W, slots, mail, tpub, done, ctas, worked, arrivals, m_at = state
    out = []
    for p, c in enumerate(ctas):
        def put(nc, **kw):
            d = dict(W=W, slots=slots, mail=mail, tpub=tpub, done=done, worked=worked,
                     arrivals=arrivals, m_at=m_at)
            d.update(kw)
            nctas = ctas[:p] + (nc,) + ctas[p + 1:]
            out.append((d["W"], d["slots"], d["mail"], d["tpub"], d["done"], nctas,
                        d["worked"], d["arrivals"], d["m_at"]))

        if c.pc == PARKED:
            if slots[p] == ASSIGNED:
                lid, g, Mp, tr = mail[p]
                if tr != g - 1:
                    raise ProtocolViolation(f"P4 transmit {tr} != WG0 state at barrier {g - 1}")
                nxt = WORK if "no_wait_gen" in bugs else WAIT_GEN
                put(Cta(nxt, lid, g, Mp), slots=slots[:p] + (ACTIVE,) + slots[p + 1:])
            elif done:
                put(Cta(EXITED))
            # else: spinning -- a self loop, no new state
        elif c.pc == WAIT_GEN:
            R = W[1]
            if R[0] == c.gen:
                if c.gen >= E:      # forked at the final barrier: termination check first
                    put(Cta(EXITED), slots=slots[:p] + (IDLE,) + slots[p + 1:])
                else:
                    put(Cta(WORK, c.lid, c.gen, c.M))
            elif R[0] > c.gen:
                raise ProtocolViolation("forked CTA missed its generation")
        elif c.pc == WORK:
            g = c.gen
            if len(m_at) <= g:
                raise ProtocolViolation(f"P1: work in interval {g} before its release")
            if g >= 1 and arrivals[g - 1] != m_at[g - 1]:
                raise ProtocolViolation(f"P1: work in interval {g} before barrier {g - 1} complete")
            if c.lid in worked[g] or not (0 <= c.lid < m_at[g]):
                raise ProtocolViolation(f"P2: id {c.lid} in interval {g} with M={m_at[g]}")
            nworked = worked[:g] + (worked[g] + (c.lid,),) + worked[g + 1:]
            ntpub = g if c.lid == 0 else tpub        # WG 0 publishes its transmit state
            put(Cta(ARRIVE, c.lid, g, c.M), worked=nworked, tpub=ntpub)
        elif c.pc == ARRIVE:
            gen, M, arr = W[0]
            if gen != c.gen:
                raise ProtocolViolation("arrived on a stale generation")
            narr = arrivals[:gen] + (arrivals[gen] + 1,) + arrivals[gen + 1:]
            if arr + 1 == M:
                mp = max(1, min(P, targets[gen] if gen < len(targets) and targets[gen] else M))
                put(Cta(SERIAL, c.lid, c.gen, c.M, 0, mp), W=((gen, M, arr + 1), W[1]), arrivals=narr)
            else:
                put(Cta(SPIN, c.lid, c.gen, c.M), W=((gen, M, arr + 1), W[1]), arrivals=narr)
        elif c.pc == SPIN:
            gen, M = W[1]
            if gen == c.gen:
                continue                                  # spin
            killed = (c.lid >= M) if "kill_by_M_only" in bugs else (gen != c.gen + 1 or c.lid >= M)
            if killed:
                if c.lid < min(c.M, m_at[c.gen + 1] if len(m_at) > c.gen + 1 else c.M):
                    raise ProtocolViolation("P3: survivor-prefix id killed")
                put(Cta(KILLED, c.lid, c.gen, c.M))
            else:
                if gen >= E:
                    put(Cta(EXITED), done=done or c.lid == 0,
                        slots=slots[:p] + (IDLE,) + slots[p + 1:])
                else:
                    put(Cta(WORK, c.lid, gen, M))
        elif c.pc == SERIAL:
            M, mp = W[0][1], c.mprime
            nid = M + c.claim_next
            if nid < mp:
                # claim one IDLE slot by CAS (each slot a separate atomic => each choice a transition)
                for q in range(P):
                    if slots[q] == IDLE:
                        ns = slots[:q] + (ASSIGNED,) + slots[q + 1:]
                        nm = mail[:q] + ((nid, c.gen + 1, mp, tpub),) + mail[q + 1:]
                        put(Cta(SERIAL, c.lid, c.gen, c.M, c.claim_next + 1, mp), slots=ns, mail=nm)
                # no IDLE slot: wait (scripted policy waits for killed CTAs to park)
            else:
                put(Cta(RELEASE, c.lid, c.gen, c.M, c.claim_next, mp))
        elif c.pc == RELEASE:       # reset the arrival word for generation g+1
            put(Cta(RELEASE_R, c.lid, c.gen, c.M, c.claim_next, c.mprime), W=((c.gen + 1, c.mprime, 0), W[1]))
        elif c.pc == RELEASE_R:     # release: publish (g+1, M') on R
            g = c.gen
            ng = g + 1
            nW = (W[0], (ng, c.mprime))
            nworked = worked + ((),) if len(worked) <= ng else worked
            narr = arrivals + (0,) if len(arrivals) <= ng else arrivals
            nm_at = m_at + (c.mprime,) if len(m_at) <= ng else m_at
            if c.lid >= c.mprime:
                put(Cta(KILLED, c.lid, g, c.M), W=nW, worked=nworked, arrivals=narr, m_at=nm_at)
            elif ng >= E:
                put(Cta(EXITED), W=nW, worked=nworked, arrivals=narr, m_at=nm_at,
                    done=done or c.lid == 0, slots=slots[:p] + (IDLE,) + slots[p + 1:])
            else:
                put(Cta(WORK, c.lid, ng, c.mprime), W=nW, worked=nworked, arrivals=narr, m_at=nm_at)
        elif c.pc == KILLED:
            put(Cta(PARKED), slots=slots[:p] + (IDLE,) + slots[p + 1:])
    return out


def explore(P: int, M0: int, targets: list[int], episodes: int, max_states: int = 2_000_000,
            bugs=frozenset()):
    """Explore every interleaving; return (n_states, n_terminal).  Raises
    ProtocolViolation on any property failure (P1-P5).

    ``bugs`` injects known-wrong protocol variants (used by the tests to show
    the model is not vacuous): "kill_by_M_only" decides a waiter's fate from
    R.M alone, ignoring that R may already be a later generation;
    "no_wait_gen" lets a forked CTA start before the release of R."""
    init = _initial(P, M0)
    seen = {init}
    q = deque([init])
    terminal = 0
    while q:
        s = q.popleft()
        succ = _successors(s, targets, P, episodes, bugs)
        if not succ:
            W, slots, mail, tpub, done, ctas, worked, arrivals, m_at = s
            if not all(c.pc == EXITED for c in ctas):
                raise ProtocolViolation(f"P5 deadlock/livelock: {ctas}")
            # P2 completeness: every interval g had exactly the ids [0, M_g)
            for g in range(episodes):
                if sorted(worked[g]) != list(range(m_at[g])):
                    raise ProtocolViolation(f"P2: interval {g} ids {worked[g]} != [0,{m_at[g]})")
            terminal += 1
            continue
        for n in succ:
            if n not in seen:
                seen.add(n)
                if len(seen) > max_states:
                    raise RuntimeError("state budget exceeded")
                q.append(n)
    return len(seen), terminal
