"""Diagnose the NCCL data plane on one GPU: partitioned BFS with P=1 at several grid sizes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import graphgen as gg
from oracle import textbook as tb
from paper_1707_01989_b200 import coop, partitioned as pt
coop.load()
g = gg.rmat(14, seed=2)
pb = pt.PartitionedBFS(gg.partition(g, 1, 0), "cuda", exchange="nccl")
pb.E_global = g.num_edges
pb.connect_nccl()
s = gg.sample_sources(g, 1)[0]
ref = tb.bfs(g, s)
for n in [8, 64, 148, 200, 260, 280, 0]:
    t = time.time()
    try:
        lv, st = pb.run(s, threads_per_wg=512, max_wgs=n, timeout_ns=5_000_000_000)
        ok = np.array_equal(lv[: g.num_vertices].cpu().numpy(), ref)
        print("max_wgs", n, "ok" if ok else "MISMATCH", f"{time.time()-t:.3f}s", st.levels, flush=True)
    except Exception as e:
        print("max_wgs", n, "ERR", e, f"{time.time()-t:.3f}s", flush=True)
pb.close()
