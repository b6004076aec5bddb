"""Small configuration sweeps on the GPU box (prints one JSON line per point)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import graphgen as gg  # noqa: E402
from paper_1707_01989_b200 import coop  # noqa: E402

if os.environ.get("COOP_LIB"):
    coop.load(os.path.abspath(os.environ["COOP_LIB"]))


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), r


what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("all", "rtt"):
    print(json.dumps({"l2_atomic_rtt_ns": coop.l2_atomic_rtt(200000)}), flush=True)
if what in ("all", "barrier"):
    for n in (148, 296, 592, 1184):
        for plain in (True, False):
            r = coop.barrier_bench(n, 100000, threads=128, plain=plain, resize_prob=0 if plain else 1 / 64)
            print(json.dumps({"barrier_ctas": n, "plain": plain, **r}), flush=True)
if what in ("all", "sssp"):
    g = gg.with_weights(gg.grid(2048, 2048, device="cuda"), seed=1)
    g.max_weight = 1000
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
    deltas = [int(x) for x in os.environ.get("DELTAS", "0,250,500,1000,2000,4000,8000").split(",")]
    for threads in (512, 1024):
        for n in (16, 74, 148):
            for delta in deltas:
                try:
                    t, (_, st) = timed(lambda: coop.sssp(g, 0, out, threads_per_wg=threads, max_wgs=n,
                                                         sssp_delta=delta), reps=2)
                except coop.CoopError as e:
                    print(json.dumps({"sssp": True, "threads": threads, "N": n, "delta": delta, "err": str(e)}),
                          flush=True)
                    continue
                print(json.dumps({"sssp": True, "threads": threads, "N": n, "delta": delta, "ms": t,
                                  "rounds": st.levels, "episodes": st.episodes, "frontier_total": st.frontier_total,
                                  "edges": st.edges_scanned, "us_per_episode": t * 1e3 / max(1, st.episodes)}),
                      flush=True)
if what in ("all", "bfs"):
    g = gg.rmat(24, seed=1, device="cuda", chunk=1 << 26)
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
    srcs = gg.sample_sources(g, 4, seed=2)
    for flags in (coop.FLAG_DIROPT, 0):
        for threads in (256, 512, 1024):
            ts = []
            for s in srcs:
                t, (_, st) = timed(lambda: coop.bfs(g, s, out, threads_per_wg=threads, flags=flags), reps=2)
                ts.append(t)
            print(json.dumps({"bfs": True, "flags": flags, "threads": threads, "ms": sorted(ts)[len(ts) // 2],
                              "levels": st.levels, "bu": st.bottom_up_levels}), flush=True)
if what == "c4":   # BASELINE.json configs[3]: 148-1184 CTAs, 1e6 barriers, random resizes p in {0, 1/64, 1/8}
    rtt = coop.l2_atomic_rtt(200000)
    print(json.dumps({"l2_atomic_rtt_ns": rtt}), flush=True)
    iters = int(os.environ.get("ITERS", "1000000"))
    for n in (148, 296, 444, 592, 740, 888, 1036, 1184):
        r = coop.barrier_bench(n, iters, threads=128, plain=True)
        print(json.dumps({"c4": True, "ctas": n, "p": "plain", "ns_per_barrier": r["ns_per_barrier"],
                          "ratio_to_rtt": r["ns_per_barrier"] / rtt}), flush=True)
        for pr in (0.0, 1 / 64, 1 / 8):
            r = coop.barrier_bench(n, iters, threads=128, resize_prob=pr, seed=3)
            print(json.dumps({"c4": True, "ctas": n, "p": pr, "ns_per_barrier": r["ns_per_barrier"],
                              "ratio_to_rtt": r["ns_per_barrier"] / rtt, "kills": r["kills"], "forks": r["forks"]}),
                  flush=True)
        r = coop.barrier_bench(n, iters // 10, threads=128, resize_prob=1 / 8, seed=4, check=True)
        print(json.dumps({"c4_check": True, "ctas": n, "p": 1 / 8, "iters": iters // 10, "kills": r["kills"],
                          "forks": r["forks"], "violations": r["violations"]}), flush=True)
if what in ("all", "barrier_small"):
    for n in (1, 2, 4, 8, 16, 32, 64, 148):
        r = coop.barrier_bench(n, 100000, threads=128, plain=True)
        print(json.dumps({"barrier_ctas": n, "plain": True, "ns_per_barrier": r["ns_per_barrier"]}), flush=True)
if what in ("all", "levels"):
    g = gg.rmat(24, seed=1, device="cuda", chunk=1 << 26)
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
    for s in gg.sample_sources(g, 3, seed=2):
        for flags in (coop.FLAG_DIROPT, 0):
            for rep in range(2):
                _, st = coop.bfs(g, s, out, threads_per_wg=512, flags=flags, level_cap=64)
            ends = st.level_end_ns
            per = [ends[0]] + [b - a for a, b in zip(ends, ends[1:])]
            print(json.dumps({"levels": True, "src": s, "flags": flags, "kernel_us": st.kernel_ns / 1e3,
                              "sizes": st.level_sizes, "level_us": [round(x / 1e3, 1) for x in per],
                              "bu": st.bottom_up_levels, "edges": st.edges_scanned}), flush=True)
if what == "ab":   # direction-switch thresholds (alpha, beta) on RMAT-24, mean kernel time over 8 sources
    g = gg.rmat(24, seed=1, device="cuda", chunk=1 << 26)
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
    srcs = gg.sample_sources(g, 8, seed=2)
    l2 = torch.empty(1 << 26, dtype=torch.int32, device="cuda")   # 256 MB > L2: flushed before every run
    for a in (2, 4, 8, 14, 32):
        for b in (8, 24, 64, 256):
            ks = []
            for s in srcs:
                best = None
                for rep in range(2):
                    l2.fill_(rep)
                    _, st = coop.bfs(g, s, out, threads_per_wg=512, flags=coop.FLAG_DIROPT, bfs_alpha=a, bfs_beta=b)
                    best = st.kernel_ns if best is None else min(best, st.kernel_ns)
                ks.append(best / 1e3)
            print(json.dumps({"alpha": a, "beta": b, "mean_kernel_us": round(sum(ks) / len(ks), 1),
                              "per_source_us": [round(k, 1) for k in ks]}), flush=True)
if what == "srcs":   # mean DIROPT kernel time on RMAT-24 over 8 sources (L2 flushed before every run)
    g = gg.rmat(24, seed=1, device="cuda", chunk=1 << 26)
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
    l2 = torch.empty(1 << 26, dtype=torch.int32, device="cuda")
    ks = []
    thr = int(os.environ.get("THREADS", "512"))
    for s in gg.sample_sources(g, 8, seed=2):
        best = None
        for rep in range(3):
            l2.fill_(rep)
            _, st = coop.bfs(g, s, out, threads_per_wg=thr, flags=coop.FLAG_DIROPT)
            best = st.kernel_ns if best is None else min(best, st.kernel_ns)
        ks.append(best / 1e3)
    print(json.dumps({"lib": os.environ.get("COOP_LIB", "default"), "mean_kernel_us": round(sum(ks) / len(ks), 1),
                      "per_source_us": [round(k, 1) for k in ks]}), flush=True)
