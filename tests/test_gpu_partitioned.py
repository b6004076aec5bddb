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


# ---------------- north_star's NCCL data plane (coop_bfs_part_nccl) ----------------
@pytest.mark.parametrize("diropt", [False, True])
def test_partitioned_bfs_nccl_single_rank(part, diropt):
    """The NCCL exchange path end to end on the one GPU of the box (NCCL refuses two ranks
    on one device): persistent kernel on the compute stream; per level the comm stream waits
    for `ready` (cuStreamWaitValue32), runs the in-place ncclAllGather of the slice and the
    counts, and writes `gathered` (cuStreamWriteValue32), which the kernel's second resizing
    barrier waits for.  Levels exact, also under random resizes (each rank's kernel resizes
    independently of the exchange)."""
    from paper_1707_01989_b200 import coop
    for g in (gg.rmat(14, seed=2), gg.disjoint_union(gg.grid(40, 30), gg.star(3000))):
        pb = part.PartitionedBFS(gg.partition(g, 1, 0), "cuda", exchange="nccl")
        pb.E_global = g.num_edges
        pb.connect_nccl()
        flags = coop.FLAG_DIROPT if diropt else 0
        for i, s in enumerate([0] + gg.sample_sources(g, 3)):
            kw = dict(policy=coop.POLICY_RANDOM, resize_prob=0.5, seed=i) if i % 2 else {}
            lv, st = pb.run(s, threads_per_wg=512, flags=flags, level_cap=4096, **kw)
            ref = tb.bfs(g, s)
            np.testing.assert_array_equal(lv[: g.num_vertices].cpu().numpy(), ref)
            assert st.level_sizes == tb.level_sizes(ref)
        pb.close()


_TWO_PROC = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {root!r})
import graphgen as gg
from oracle import textbook as tb
from paper_1707_01989_b200 import coop, partitioned as pt
rank = int(sys.argv[1])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=2)
torch.cuda.set_device(0)
g = gg.rmat(12, seed=7)
pb = pt.PartitionedBFS(gg.partition(g, 2, rank), "cuda")
pb.E_global = g.num_edges
pb.connect_ipc()                       # CUDA IPC handles all-gathered over torch.distributed
ok = True
for i, s in enumerate(gg.sample_sources(g, 3)):
    dist.barrier()
    lv, st = pb.run(s, threads_per_wg=256, max_wgs=8, timeout_ns=120_000_000_000,
                    flags=coop.FLAG_DIROPT if i % 2 else 0)
    ref = tb.bfs(g, s)[pb.part.v_begin:pb.part.v_end]
    ok &= bool(np.array_equal(lv[: pb.part.v_end - pb.part.v_begin].cpu().numpy(), ref))
dist.barrier()
pb.close()
print("RANK", rank, "OK" if ok else "MISMATCH", flush=True)
"""


def test_partitioned_bfs_two_processes_ipc(part, tmp_path):
    """Two OS processes (one rank each) on the box's single GPU: the exchange buffers are
    shared by CUDA IPC handles all-gathered over torch.distributed (connect_ipc), and every
    level's slice stores and .sys-scope release/acquire flags cross the process boundary --
    the same code path as across NVLink between GPUs.  The two persistent kernels belong to
    different contexts, so the GPU time-slices them (slow, but each barrier completes)."""
    import socket
    import subprocess
    import sys
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    script = tmp_path / "two.py"
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script.write_text(_TWO_PROC.format(root=root, port=port))
    procs = [subprocess.Popen([sys.executable, str(script), str(r)], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=600)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("two-process partitioned BFS timed out")
    for r, o in enumerate(outs):
        assert f"RANK {r} OK" in o, o[-3000:]


# ---------------- partitioned SSSP: (vertex, distance) exchange ----------------
@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("name", ["grid", "rmat", "disconnected"])
def test_partitioned_sssp_matches_dijkstra(part, P, name):
    g = {"grid": lambda: gg.grid(40, 37), "rmat": lambda: gg.rmat(12, seed=5),
         "disconnected": lambda: gg.disjoint_union(gg.rmat(10, seed=3), gg.path(200))}[name]()
    g = gg.with_weights(g, seed=6)
    parts = None
    for s in [0] + gg.sample_sources(g, 2):
        d, stats, parts = part.simulate_one_gpu_sssp(g, P, s, parts=parts, level_cap=4096)
        np.testing.assert_array_equal(d.cpu().numpy().view(np.uint32), tb.dijkstra(g, s))
    for pb in parts:
        pb.close()


def test_partitioned_sssp_under_resizes(part):
    from paper_1707_01989_b200 import coop
    g = gg.with_weights(gg.grid(30, 45), seed=2)
    parts = None
    for seed in range(3):
        d, stats, parts = part.simulate_one_gpu_sssp(g, 3, 7, parts=parts, ctas_per_rank=12,
                                                     policy=coop.POLICY_RANDOM, resize_prob=0.5, seed=seed,
                                                     flags=coop.FLAG_CHECK)
        np.testing.assert_array_equal(d.cpu().numpy().view(np.uint32), tb.dijkstra(g, 7))
        assert sum(st.kills + st.forks for st in stats) > 0
    for pb in parts:
        pb.close()
