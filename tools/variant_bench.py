"""A/B timing of libcoop build variants on RMAT-24 (one subprocess per variant .so).

    python tools/variant_bench.py build_variants/a.so build_variants/b.so ...
Per variant: cooperative BFS (NEVER) and the non-cooperative kernel (BARRIER_PLAIN),
direction-optimising, 512 threads, N-1 workers, 8 sources x 3 reps (CUDA events,
L2 flushed); prints one JSON line per variant with median kernel-call ms."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, statistics, sys, torch
sys.path.insert(0, %r)
import graphgen as gg
from paper_1707_01989_b200 import coop
coop.load(os.path.abspath(sys.argv[1]))
g = gg.rmat(int(os.environ.get("SCALE", "24")), seed=1, device="cuda", chunk=1 << 26)
coop._bfs_csr(g)
srcs = gg.sample_sources(g, 8, seed=2)
out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
N = coop.device_query(0, 512)["max_coresident"] - 1
arms = {"coop_never": {}, "noncoop": dict(barrier_mode=coop.BARRIER_PLAIN),
        "coop_armed": dict(policy=coop.POLICY_SCHEDULER)}
res = {a: [] for a in arms}
for s in srcs:
    for rep in range(4):
        for a, kw in arms.items():
            flush.fill_(rep)
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record(); k1.record()
            coop.bfs(g, s, out, threads_per_wg=512, max_wgs=N, flags=coop.FLAG_DIROPT,
                     ev_kernel_start=k0, ev_kernel_end=k1, **kw)
            torch.cuda.synchronize()
            if rep:
                res[a].append(k0.elapsed_time(k1))
print(json.dumps({"lib": sys.argv[1], **{a: round(statistics.median(v), 4) for a, v in res.items()}}), flush=True)
""" % ROOT

for lib in sys.argv[1:]:
    r = subprocess.run([sys.executable, "-c", CHILD, lib], capture_output=True, text=True, timeout=600)
    print(r.stdout.strip() or json.dumps({"lib": lib, "err": r.stderr[-2000:]}), flush=True)
