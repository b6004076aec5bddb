"""Barrier phase breakdown (needs a -DCOOP_TRACE=1 build): python tools/barrier_trace.py LIB"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_01989_b200 import coop
coop.load(os.path.abspath(sys.argv[1]))
names = ["entry_sync", "arrival", "wait_release", "serial_exit", "interval"]
for n in (1, 2, 148, 1184):
    r = coop.barrier_bench(n, 20000, threads=128, plain=True)
    t = coop.debug_trace()
    res = {"ctas": n, "ns_per_barrier": round(r["ns_per_barrier"], 1)}
    for role, o in (("waiter", 0), ("last", 8)):
        cnt = t[o + 5]
        if cnt:
            res[role] = {k: round(t[o + i] / cnt, 1) for i, k in enumerate(names)}
            res[role]["count"] = cnt
    print(json.dumps(res), flush=True)
