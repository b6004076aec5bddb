"""O3: brute-force enumeration of schedules on tiny graphs (TEST INFRASTRUCTURE ONLY).

BASELINE.json north_star: "results independent of any kill/fork schedule,
found by brute-force enumeration of schedules on tiny graphs".  Two axes:

* ``all_resize_sequences`` -- every target sequence M'_e in [1, N]^E over the
  E resizing-barrier episodes (the scheduler's choices);
* ``all_interleavings`` -- every interleaving of thread steps and
  workgroup-level primitives (stateless DFS over the chooser's decisions, the
  nondeterminism of rule Thread-Step).

Each run goes through :mod:`oracle.coop_sim` and is returned to the caller,
which compares it with the textbook oracle.
"""
from __future__ import annotations

import itertools
from typing import Callable, Iterator

from . import coop_sim as cs


def all_resize_sequences(g, source, *, N: int, d: int = 1, mode: str = "bfs",
                         episodes: int | None = None, chooser_seed: int = 0) -> Iterator[tuple[tuple, cs.SimResult]]:
    """Yield (sequence, result) for every M' sequence in [1,N]^episodes."""
    if episodes is None:
        episodes = len(cs.simulate(g, source, mode=mode, N=N, d=d).episodes)
    for seq in itertools.product(range(1, N + 1), repeat=episodes):
        r = cs.simulate(g, source, mode=mode, N=N, d=d,
                        scheduler=cs.SequenceScheduler(list(seq)),
                        chooser=cs.RandomChooser(chooser_seed))
        yield seq, r


def all_interleavings(g, source, *, N: int, d: int = 1, mode: str = "bfs",
                      scheduler_factory: Callable[[], cs.Scheduler] = cs.NeverResize,
                      preemption_bound: int | None = None,
                      max_runs: int = 200_000) -> Iterator[cs.SimResult]:
    """Exhaustive DFS over every choice point of the interleaver.

    Stateless model checking: re-run from the initial state with a choice
    prefix; after each run advance the deepest choice with an untried branch.
    With ``preemption_bound`` = K only schedules with at most K preemptions
    (switching away from a thread that could continue) are explored -- every
    schedule within the bound is run.  Raises RuntimeError if more than
    ``max_runs`` runs would be needed.
    """
    prefix: list[int] = []
    runs = 0
    while True:
        ch = cs.ReplayChooser(prefix)
        r = cs.simulate(g, source, mode=mode, N=N, d=d, scheduler=scheduler_factory(), chooser=ch)
        yield r
        runs += 1
        if runs > max_runs:
            raise RuntimeError("interleaving budget exceeded")
        trace = ch.trace
        pre = [0]
        for c, _, cont in trace:
            pre.append(pre[-1] + (1 if (cont and c > 0) else 0))
        pos = len(trace) - 1
        while pos >= 0:
            c, n, cont = trace[pos]
            if c + 1 < n:
                cost = pre[pos] + (1 if cont else 0)
                if preemption_bound is None or cost <= preemption_bound:
                    break
            pos -= 1
        if pos < 0:
            return
        prefix = [c for c, _, _ in trace[:pos]] + [trace[pos][0] + 1]
