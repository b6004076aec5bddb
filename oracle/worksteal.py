"""O6: cooperative work stealing workload (TEST INFRASTRUCTURE, NOT PRODUCT CODE).

Fig. 2 of the paper is a work-stealing kernel whose tasks
"may lead to new tasks being created"; §3.2 adapts it to the
cooperative model with ``offer_kill`` / ``request_fork`` at the head of the
main loop.  The paper names no concrete task set (its octree /
game-tree apps are not reproduced), so the workload is a seeded
implicit task tree (reading R19):

* root task ``(id = seed, depth = 0)``;
* ``h = splitmix64(id)``;
* children: none at ``depth == D``; else ``B`` (``fixed``) or ``(h >> 32) % (B + 1)``;
  child ``j`` is ``(h + j + 1 mod 2^64, depth + 1)``;
* the task's value is ``sum_{l < TW} chain(h ^ l, R) mod 2^64`` where
  ``chain(x, R)`` applies splitmix64 ``R`` times (the task's "work",
  P:376 ``process_task``).

What the kernel must reproduce is schedule independent: the number of tasks,
the histogram of tasks per depth and the 64-bit wrapping sum of the values,
whatever workgroup pops or steals what and whoever is killed or forked.

Pins (tests/test_oracle_worksteal.py): splitmix64's published first output
for state 0; closed forms of fixed-fanout trees (B^d tasks at depth d);
degenerate trees (D = 0, B = 0, fanout 1 chains); the value of a task with
R = 0 / TW = 1; and equality of two traversal orders (stack vs level by level).
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
TW = 256          # lanes of work per task (R19)


def splitmix64(x: int) -> int:
    """splitmix64 output function (Steele, Lea, Flood 2014) of the state x."""
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _splitmix64_vec(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def task_value(task_id: int, rounds: int, tw: int = TW) -> int:
    """value(t) = sum over lanes l < tw of chain(h ^ l, rounds), mod 2^64."""
    h = splitmix64(task_id)
    x = np.uint64(h) ^ np.arange(tw, dtype=np.uint64)
    for _ in range(rounds):
        x = _splitmix64_vec(x)
    return int(x.sum(dtype=np.uint64)) & M64


def children(task_id: int, depth: int, D: int, B: int, fixed: bool):
    if depth >= D:
        return []
    h = splitmix64(task_id)
    n = B if fixed else (h >> 32) % (B + 1)
    return [((h + j + 1) & M64, depth + 1) for j in range(n)]


def run_stack(seed: int, D: int, B: int, fixed: bool = False, rounds: int = 0, tw: int = TW,
              max_tasks: int = 1 << 22):
    """Fig. 2's loop with one queue: pop a task, process it, push its children."""
    stack = [(seed & M64, 0)]
    count, total = 0, 0
    hist = [0] * (D + 1)
    while stack:
        tid, d = stack.pop()
        count += 1
        if count > max_tasks:
            raise ValueError("task tree larger than max_tasks")
        hist[d] += 1
        total = (total + task_value(tid, rounds, tw)) & M64
        stack.extend(children(tid, d, D, B, fixed))
    return {"count": count, "total": total, "hist": hist}


def run_levels(seed: int, D: int, B: int, fixed: bool = False, rounds: int = 0, tw: int = TW):
    """The same tree expanded level by level (a different traversal order)."""
    level = [(seed & M64, 0)]
    count, total = 0, 0
    hist = [0] * (D + 1)
    while level:
        nxt = []
        for tid, d in level:
            count += 1
            hist[d] += 1
            total = (total + task_value(tid, rounds, tw)) & M64
            nxt.extend(children(tid, d, D, B, fixed))
        level = nxt
    return {"count": count, "total": total, "hist": hist}
