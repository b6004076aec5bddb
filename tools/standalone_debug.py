import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import graphgen as gg
from paper_1707_01989_b200 import coop
g = gg.rmat(24, seed=1, device="cuda", chunk=1 << 26)
s = gg.sample_sources(g, 1, seed=2)[0]
out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
info = coop.device_query(0, 256)
N = info["max_coresident"] - 1
for label, kw in [("default", {}), ("maxN", {"max_wgs": N}), ("maxN_dopt", {"max_wgs": N, "flags": 2}),
                  ("dopt", {"flags": 2}), ("sched_notask", {"flags": 2, "policy": 3}),
                  ("maxN_dopt_again", {"max_wgs": N, "flags": 2})]:
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record()
        _, st = coop.bfs(g, s, out, threads_per_wg=256, **kw)
        e1.record(); torch.cuda.synchronize()
        print(json.dumps({"label": label, "rep": rep, "ev_ms": e0.elapsed_time(e1), "wall_ms": 1e3 * (time.perf_counter() - t0), "kernel_ms": st.kernel_ns / 1e6, "n_wgs": st.n_wgs}), flush=True)
