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
if os.environ.get("VB_TD"):
    arms["topdown_never"] = dict(flags=0)
res = {a: [] for a in arms}
for s in srcs:
    for rep in range(4):
        for a, kw in arms.items():
            flush.fill_(rep)
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record(); k1.record()
            kw2 = dict(kw)
            fl = kw2.pop("flags", coop.FLAG_DIROPT)
            coop.bfs(g, s, out, threads_per_wg=512, max_wgs=N, flags=fl,
                     ev_kernel_start=k0, ev_kernel_end=k1, **kw2)
            torch.cuda.synchronize()
            if rep:
                res[a].append(k0.elapsed_time(k1))
print(json.dumps({"lib": sys.argv[1], **{a: round(statistics.median(v), 4) for a, v in res.items()}}), flush=True)
""" % ROOT

CHILD_SSSP = r"""
import json, os, statistics, sys, torch
sys.path.insert(0, %r)
import graphgen as gg
from paper_1707_01989_b200 import coop
coop.load(os.path.abspath(sys.argv[1]))
g = gg.with_weights(gg.grid(2048, 2048, device="cuda"), seed=1)
g.max_weight = 1000
out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
res = {}
for delta in [int(x) for x in os.environ.get("DELTAS", "0,64000").split(",")]:
    for thr in (256, 512):
        ts = []
        for rep in range(3):
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record(); k1.record()
            _, st = coop.sssp(g, 0, out, threads_per_wg=thr, max_wgs=148, sssp_delta=delta,
                              ev_kernel_start=k0, ev_kernel_end=k1)
            torch.cuda.synchronize()
            ts.append(k0.elapsed_time(k1))
        ms = statistics.median(ts)
        res[f"d{delta}_t{thr}"] = {"ms": round(ms, 3), "episodes": st.episodes,
                                   "us_per_ep": round(ms * 1e3 / st.episodes, 2), "relaxed": st.edges_scanned}
print(json.dumps({"lib": sys.argv[1], **res}), flush=True)
""" % ROOT

CHILD_BAR = r"""
import json, os, sys, numpy as np, torch
sys.path.insert(0, %r)
import graphgen as gg
from oracle import textbook as tb
from paper_1707_01989_b200 import coop
coop.load(os.path.abspath(sys.argv[1]))
res = {"rtt_ns": round(coop.l2_atomic_rtt(200000), 1)}
for n in (148, 592, 1184):
    a = coop.barrier_bench(n, 200000, threads=128, plain=True)
    b = coop.barrier_bench(n, 200000, threads=128, resize_prob=1 / 64, seed=3)
    c = coop.barrier_bench(n, 50000, threads=128, resize_prob=1 / 8, seed=4, check=True)
    res[str(n)] = {"plain": round(a["ns_per_barrier"], 1), "p64": round(b["ns_per_barrier"], 1),
                   "chk_violations": c.get("violations")}
g = gg.rmat(16, seed=5); gd = g.to("cuda")
ok = True
for s in gg.sample_sources(g, 4):
    for kw in (dict(flags=coop.FLAG_DIROPT), dict(flags=coop.FLAG_CHECK, policy=coop.POLICY_RANDOM, resize_prob=0.5, seed=s)):
        lv, _ = coop.bfs(gd, s, **kw)
        ok &= bool(np.array_equal(lv.cpu().numpy(), tb.bfs(g, s)))
res["bfs_parity"] = ok
print(json.dumps({"lib": sys.argv[1], **res}), flush=True)
""" % ROOT

if os.environ.get("VB_MODE") == "sssp":
    CHILD = CHILD_SSSP
elif os.environ.get("VB_MODE") == "barrier":
    CHILD = CHILD_BAR

for lib in sys.argv[1:]:
    r = subprocess.run([sys.executable, "-c", CHILD, lib], capture_output=True, text=True, timeout=600)
    print(r.stdout.strip() or json.dumps({"lib": lib, "err": r.stderr[-2000:]}), flush=True)
