"""Kernel-level preemption overhead model (TEST INFRASTRUCTURE ONLY).

PAPER.md:1286-1292 (§5.5): a graphics task of period P and duration D
preempting a whole compute kernel costs an overhead factor P / (P - D).
Table 3 lists 1.04 / 1.08 / 1.33 for the light (70, 3),
medium (40, 3) and heavy (40, 10) presets.
"""

PRESETS_MS = {"light": (70.0, 3.0), "medium": (40.0, 3.0), "heavy": (40.0, 10.0)}


def preemption_overhead(P: float, D: float) -> float:
    if not (0 <= D < P):
        raise ValueError("need 0 <= D < P")
    return P / (P - D)
