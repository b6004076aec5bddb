"""A/B the barrier implementation switches (coop_rt.cuh COOP_* macros).

    python tools/barrier_variants.py build_variants/libcoop_X.so ...
Each library runs in its own subprocess: barrier ns at 148 / 1184 CTAs (plain
and resizing with the message-passing check) and a BFS parity spot check.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys
sys.path.insert(0, %(root)r)
import numpy as np, torch
from paper_1707_01989_b200 import coop
coop.load(%(lib)r)
import graphgen as gg
from oracle import textbook as tb
res = {"lib": %(lib)r}
for n in (148, 1184):
    a = coop.barrier_bench(n, 100000, threads=128, plain=True)
    b = coop.barrier_bench(n, 100000, threads=128, resize_prob=1/16, seed=3, check=True)
    res[f"plain_{n}"] = round(a["ns_per_barrier"], 1)
    res[f"resize_check_{n}"] = round(b["ns_per_barrier"], 1)
    res[f"violations_{n}"] = b["violations"]
g = gg.rmat(16, seed=1)
gd = g.to("cuda")
ok = True
for s in gg.sample_sources(g, 3):
    for flags in (0, coop.FLAG_DIROPT):
        lv, _ = coop.bfs(gd, s, flags=flags | coop.FLAG_CHECK, policy=coop.POLICY_RANDOM, resize_prob=0.5, seed=s)
        ok &= bool(np.array_equal(lv.cpu().numpy(), tb.bfs(g, s)))
res["bfs_parity"] = ok
print(json.dumps(res), flush=True)
'''

for lib in sys.argv[1:]:
    r = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT, "lib": os.path.abspath(lib)}],
                       capture_output=True, text=True, timeout=600)
    out = [l for l in r.stdout.splitlines() if l.startswith("{")]
    print(out[-1] if out else json.dumps({"lib": lib, "error": r.stderr[-500:]}), flush=True)
