"""Profiling driver: RMAT-`scale` cooperative BFS, `warm` untimed calls then `n` calls.

Used under ncu on the GPU box (one process, one GPU), e.g.
    ncu --set full --clock-control none --import-source on -k regex:coop_kernel -s 2 -c 1 \
        -o gpurun_out/prof python tools/prof_bfs.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import graphgen as gg  # noqa: E402
from paper_1707_01989_b200 import coop  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--warm", type=int, default=2)
ap.add_argument("--n", type=int, default=1)
ap.add_argument("--threads", type=int, default=512)
ap.add_argument("--app", default="bfs")
ap.add_argument("--flags", type=int, default=2, help="2 = COOP_FLAG_DIROPT, 0 = top-down")
ap.add_argument("--policy", default="never", help="never | scheduler (the armed arm: scheduler CTA, no task)")
ap.add_argument("--src", type=int, default=-1, help="fixed source index (default: cycle over 8)")
args = ap.parse_args()

dev = torch.device("cuda", 0)
if args.app == "bfs":
    g = gg.rmat(args.scale, seed=1, device=dev, chunk=1 << 26)
    srcs = gg.sample_sources(g, 8, seed=2)
    out = torch.empty(g.num_vertices, dtype=torch.int32, device=dev)
    for i in range(args.warm + args.n):
        kw = dict(policy=coop.POLICY_SCHEDULER) if args.policy == "scheduler" else {}
        N = coop.device_query(0, args.threads)["max_coresident"] - 1
        s = srcs[args.src] if args.src >= 0 else srcs[i % 8]
        _, st = coop.bfs(g, s, out, threads_per_wg=args.threads, flags=args.flags, max_wgs=N, **kw)
        print(f"call {i}: kernel_ms={st.kernel_ns / 1e6:.3f} edges={st.edges_scanned} levels={st.levels}", flush=True)
else:
    g = gg.with_weights(gg.grid(2048, 2048, device=dev), seed=1)
    g.max_weight = 1000
    out = torch.empty(g.num_vertices, dtype=torch.int32, device=dev)
    for i in range(args.warm + args.n):
        _, st = coop.sssp(g, 0, out, threads_per_wg=256, max_wgs=148)
        print(f"call {i}: kernel_ms={st.kernel_ns / 1e6:.3f} rounds={st.levels}", flush=True)
