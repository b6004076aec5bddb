"""Multitasking experiment grid -- the analogue of the paper's Fig. 5 / Fig. 6
 on B200.

A cooperative BFS runs while the in-kernel scheduler CTA posts a competing
non-cooperative task every P; each instance demands Q workgroups and carries
N blocks of E each (total work E on all N workgroups, so ~ceil(N/Q)*E on Q:
"the more workgroups are allocated ... the faster it can compute").
Presets are the paper's light/medium/heavy (P, E) = (70,3)/(40,3)/(40,10) ms
 scaled by `--scale-time` so that several instances fall inside
one traversal.  Q in {1, N/4, N/2, N-1}; barrier in {query,
naive}.  Graphs: 2-D grid (deep, the "USA road" role) and RMAT
(wide, the "rmat" / "G3_circuit" role).

Reported per point: cooperative slowdown vs standalone, mean/p99 gather time
(demand -> last surrender), kill latency (demand -> first task block
start), task execution time, achieved period.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import graphgen as gg  # noqa: E402
from paper_1707_01989_b200 import coop  # noqa: E402

PRESETS_MS = {"light": (70.0, 3.0), "medium": (40.0, 3.0), "heavy": (40.0, 10.0)}


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), r


def pct(v, q):
    v = sorted(v)
    return v[min(len(v) - 1, int(q * len(v)))] if v else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--graphs", default="grid,rmat")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--threads", type=int, default=256)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    info = coop.device_query(0, args.threads)
    N = info["max_coresident"] - 1                       # one slot is the scheduler CTA
    graphs = {}
    if "grid" in args.graphs:
        graphs["grid2048"] = (gg.grid(2048, 2048, device="cuda"), 0, 0, 1 / 10.0)
    if "rmat" in args.graphs:
        g = gg.rmat(24, seed=1, device="cuda", chunk=1 << 26)
        graphs["rmat24"] = (g, gg.sample_sources(g, 1, seed=2)[0], coop.FLAG_DIROPT, 1 / 100.0)
    rows = []
    for gname, (g, src, flags, tscale) in graphs.items():
        out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
        coop.bfs(g, src, out, threads_per_wg=args.threads, flags=flags, max_wgs=N)   # warm-up (graph caching)
        base = [timed(lambda: coop.bfs(g, src, out, threads_per_wg=args.threads, flags=flags,
                                       max_wgs=N))[0] for _ in range(args.reps)]
        t_alone = statistics.median(base)
        rows.append({"graph": gname, "standalone_ms": t_alone, "N": N})
        print(json.dumps(rows[-1]), flush=True)
        for preset, (P_ms, E_ms) in PRESETS_MS.items():
            P_ns, E_ns = int(P_ms * tscale * 1e6), int(E_ms * tscale * 1e6)
            for q in sorted({1, max(1, N // 4), max(1, N // 2), N - 1}):
                for mode, bm in (("query", coop.BARRIER_QUERY), ("naive", coop.BARRIER_NAIVE)):
                    ts, gather, lat, exe, ends, posted, done = [], [], [], [], [], 0, 0
                    for _ in range(args.reps):
                        t, (_, st) = timed(lambda: coop.bfs(
                            g, src, out, threads_per_wg=args.threads, flags=flags, barrier_mode=bm,
                            policy=coop.POLICY_SCHEDULER, task_wgs=q, task_blocks=N, task_block_ns=E_ns,
                            task_period_ns=P_ns, task_first_ns=P_ns // 4, event_cap=4096))
                        ts.append(t)
                        posted += st.tasks_posted
                        done += st.tasks_completed
                        ev = [e for e in st.task_events if e["t_end"]]
                        for e in ev:
                            if e["t_last_surrender"]:
                                gather.append((e["t_last_surrender"] - e["t_arrive"]) / 1e3)
                            if e["t_first_start"]:
                                lat.append((e["t_first_start"] - e["t_arrive"]) / 1e3)
                                exe.append((e["t_end"] - e["t_first_start"]) / 1e3)
                        e_sorted = sorted(e["t_end"] for e in ev)
                        ends.extend((b - a) / 1e3 for a, b in zip(e_sorted, e_sorted[1:]))
                    periods = ends
                    row = {"graph": gname, "preset": preset, "P_us": P_ns / 1e3, "E_us": E_ns / 1e3, "Q": q,
                           "barrier": mode, "coop_ms": statistics.median(ts),
                           "slowdown": statistics.median(ts) / t_alone,
                           "tasks_posted": posted, "tasks_completed": done,
                           "gather_us_mean": statistics.mean(gather) if gather else None,
                           "gather_us_p99": pct(gather, 0.99),
                           "kill_latency_us_p50": pct(lat, 0.5), "kill_latency_us_p99": pct(lat, 0.99),
                           "exec_us_mean": statistics.mean(exe) if exe else None,
                           "period_us_median": statistics.median(periods) if periods else None}
                    rows.append(row)
                    print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
