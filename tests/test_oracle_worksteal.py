"""Pins of the work-stealing oracle O6 (oracle/worksteal.py) -- CPU only."""
import numpy as np
import pytest

from oracle import worksteal as ws


def test_splitmix64_published_vector():
    # SplitMix64 seeded with state 0: the first output is 0xE220A8397B1DCDAF
    # (the reference sequence of Steele, Lea, Flood 2014 / java.util.SplittableRandom)
    assert ws.splitmix64(0) == 0xE220A8397B1DCDAF
    # the second output is the function of state 2 * golden gamma
    assert ws.splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def test_value_special_cases():
    h = ws.splitmix64(12345)
    # R = 0, one lane: the value is h itself
    assert ws.task_value(12345, 0, tw=1) == h
    # R = 0: sum of h ^ l
    assert ws.task_value(12345, 0, tw=4) == sum(h ^ l for l in range(4)) & ws.M64
    # R = 1, one lane: one application
    assert ws.task_value(12345, 1, tw=1) == ws.splitmix64(h)
    # R = 2 composes
    assert ws.task_value(7, 2, tw=1) == ws.splitmix64(ws.splitmix64(ws.splitmix64(7)))


@pytest.mark.parametrize("B,D", [(2, 6), (3, 4), (1, 9), (5, 2)])
def test_fixed_fanout_closed_form(B, D):
    r = ws.run_stack(11, D, B, fixed=True)
    assert r["hist"] == [B ** d for d in range(D + 1)]
    n = D + 1 if B == 1 else (B ** (D + 1) - 1) // (B - 1)
    assert r["count"] == n


def test_degenerate_trees():
    r = ws.run_stack(5, 0, 4)
    assert r["count"] == 1 and r["hist"] == [1]
    assert r["total"] == ws.task_value(5, 0)
    r = ws.run_stack(5, 7, 0)
    assert r["count"] == 1 and r["hist"] == [1] + [0] * 7


def test_traversal_order_independent():
    for seed in (1, 2, 3):
        a = ws.run_stack(seed, 10, 4, rounds=2, tw=8)
        b = ws.run_levels(seed, 10, 4, rounds=2, tw=8)
        assert a == b
        assert a["count"] == sum(a["hist"])


def test_random_tree_fanout_distribution():
    # the fanout draw (h >> 32) % (B + 1) is uniform on [0, B]: mean B/2 over many tasks
    fan = [(ws.splitmix64(i) >> 32) % 5 for i in range(20000)]
    assert abs(np.mean(fan) - 2.0) < 0.05
