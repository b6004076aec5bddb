"""GPU parity of the 1-D partitioned cooperative BFS (configs[4]).  The box has
one GPU, so P ranks run as P concurrent cooperative kernels on it (separate
streams and workspaces) exchanging frontiers through plain device pointers --
the same kernel code path as NVLink peer memory, only the addresses differ."""
import numpy as np
import pytest
import torch

import graphgen as gg
from oracle import textbook as tb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def part():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1707_01989_b200 import build, partitioned as pt
    build.build()
    return pt


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("name", ["rmat12", "grid", "disconnected", "star"])
def test_partitioned_bfs_matches_textbook(part, P, name):
    g = {"rmat12": lambda: gg.rmat(12, seed=1), "grid": lambda: gg.grid(50, 70),
         "disconnected": lambda: gg.disjoint_union(gg.rmat(10, seed=3), gg.path(100)),
         "star": lambda: gg.star(20000)}[name]()
    parts = None
    for s in [0] + gg.sample_sources(g, 2):
        lv, stats, parts = part.simulate_one_gpu(g, P, s, threads=256, ctas_per_rank=16, parts=parts, level_cap=4096)
        ref = tb.bfs(g, s)
        np.testing.assert_array_equal(lv.cpu().numpy(), ref)
        assert stats[0].level_sizes == tb.level_sizes(ref)
        assert sum(st.reached for st in stats) == int((ref >= 0).sum())
    for pb in parts:
        pb.close()


def test_partitioned_hubs_and_resizes(part):
    """Static hubs (local degree >= hub_degree) take the edge-balanced path; each
    rank resizes independently under a random schedule."""
    g = gg.disjoint_union(gg.star(30000), gg.rmat(11, seed=4))
    P = 2
    parts = [part.PartitionedBFS(gg.partition(g, P, r), "cuda", hub_degree=256) for r in range(P)]
    assert all(pb.hub_ids.numel() >= 1 for pb in parts)
    from paper_1707_01989_b200 import coop
    for seed, s in enumerate([0, 5, 30001]):
        lv, stats, _ = part.simulate_one_gpu(g, P, s, threads=256, ctas_per_rank=24, parts=parts,
                                             policy=coop.POLICY_RANDOM, resize_prob=0.6, seed=seed,
                                             flags=coop.FLAG_CHECK)
        np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(g, s))
    for pb in parts:
        pb.close()


def test_partitioned_rmat_partition_generator(part):
    """Per-rank generation (graphgen.rmat_partition, on the GPU) == partition of
    the full graph, and the partitioned BFS over it matches the textbook BFS."""
    P, scale = 4, 13
    g = gg.rmat(scale, seed=2)
    parts = []
    for r in range(P):
        p1 = gg.rmat_partition(scale, P, r, seed=2, device="cuda")
        p0 = gg.partition(g, P, r)
        assert torch.equal(p1.row_offsets.cpu(), p0.row_offsets) and torch.equal(p1.col_local.cpu(), p0.col_local)
        parts.append(part.PartitionedBFS(p1, "cuda"))
    s = gg.sample_sources(g, 1)[0]
    lv, _, _ = part.simulate_one_gpu(g, P, s, threads=256, ctas_per_rank=16, parts=parts)
    np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(g, s))
    for pb in parts:
        pb.close()


@pytest.mark.parametrize("P", [1, 2, 4])
def test_partitioned_direction_optimising(part, P):
    """Bottom-up levels on the owned rows, direction chosen from the globally
    exchanged n_f / m_f: identical levels, and R-MAT triggers bottom-up."""
    from paper_1707_01989_b200 import coop
    g = gg.rmat(14, seed=6)
    parts = None
    for s in gg.sample_sources(g, 3):
        lv, stats, parts = part.simulate_one_gpu(g, P, s, threads=256, ctas_per_rank=16, parts=parts,
                                                 flags=coop.FLAG_DIROPT, level_cap=64)
        ref = tb.bfs(g, s)
        np.testing.assert_array_equal(lv.cpu().numpy(), ref)
        assert stats[0].level_sizes == tb.level_sizes(ref)
        assert len({st.bottom_up_levels for st in stats}) == 1      # same direction on every rank
        assert stats[0].bottom_up_levels >= 1
    g2 = gg.disjoint_union(gg.grid(30, 30), gg.star(3000))
    lv, _, p2 = part.simulate_one_gpu(g2, P, 0, threads=256, ctas_per_rank=16, flags=coop.FLAG_DIROPT)
    np.testing.assert_array_equal(lv.cpu().numpy(), tb.bfs(g2, 0))
    for pb in parts + p2:
        pb.close()
