"""Where the time between two back-to-back cooperative BFS kernels goes: torch.profiler
(CUPTI) timeline of pipelined coop_bfs_launch calls on RMAT-24 -- memcpy / memset /
kernel start and duration per call, and the idle gaps between them.

    python tools/call_gap_probe.py [--scale 24] [--calls 6]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import graphgen as gg  # noqa: E402
from paper_1707_01989_b200 import coop  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--calls", type=int, default=6)
args = ap.parse_args()
coop.load()
g = gg.rmat(args.scale, seed=1, device="cuda", chunk=1 << 26)
coop._bfs_csr(g)
srcs = gg.sample_sources(g, 16, seed=2)
outs = [torch.empty(g.num_vertices, dtype=torch.int32, device="cuda") for _ in range(args.calls)]


import time  # noqa: E402
host = []


def run():
    inflight = []
    t00 = time.perf_counter()
    for j in range(args.calls):
        a = time.perf_counter()
        inflight.append(coop.BfsCall(g, srcs[j], outs[j], threads_per_wg=512, flags=coop.FLAG_DIROPT, workspace=j % 2))
        b = time.perf_counter()
        host.append((f"launch {j}", (a - t00) * 1e6, (b - a) * 1e6))
        if len(inflight) == 2:
            a = time.perf_counter()
            inflight.pop(0).wait()
            b = time.perf_counter()
            host.append((f"wait {j - 1}", (a - t00) * 1e6, (b - a) * 1e6))
    for c in inflight:
        c.wait()
    torch.cuda.synchronize()


run()
host.clear()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
for name, start, dur in host:
    print(f"host {name:10s} at {start:9.1f} us  took {dur:8.1f} us")
path = "/tmp/call_gap_trace.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
ev = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
prev_end = None
for e in ev:
    gap = (e["ts"] - prev_end) if prev_end is not None else 0.0
    print(f"{e['ts'] - t0:10.1f} us  dur {e['dur']:8.1f} us  gap {gap:7.1f}  {e['cat']:11s} {e['name'][:70]}")
    prev_end = e["ts"] + e["dur"]
