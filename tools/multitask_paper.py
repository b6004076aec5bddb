"""The paper's multitasking experiment at its own presets (configs[2](iii); PAPER.md
:1045, :1061-1062, :1135-1255): the cooperative BFS runs in a loop over sources
INSIDE ONE persistent launch for >= 10 s (coop_bfs_loop) while the in-kernel
scheduler CTA posts a competing non-cooperative task every P ms whose total work
is E ms on all N workgroups (blocks of E/10 each, so it takes ~E*N/Q on Q
workgroups: "the more workgroups ... the faster").

Presets (P, E) = light (70, 3), medium (40, 3), heavy (40, 10) ms;
Q in {1, N/4, N/2, N-1}; resizing barrier in {query, naive}
(P:1145-1146).  Reported per cell: multitasked GTEPS (Graph500 edges of the
runs / loop time), slowdown vs the standalone loop, kill latency p50/p99
(demand posted -> first task block starts), gather p50/p99 (-> last workgroup
surrendered), task execution time, achieved period,
and the last run's levels compared with the oracle.

    python tools/multitask_paper.py [--scale 24] [--loop-s 10] [--cells all|bench]
"""
import argparse
import json
import os
import statistics
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PRESETS_MS = {"light": (70.0, 3.0), "medium": (40.0, 3.0), "heavy": (40.0, 10.0)}


def pct(v, q):
    v = sorted(v)
    return v[min(len(v) - 1, int(q * len(v)))] if v else None


class MultitaskRunner:
    """Shared by this tool and bench.py's extras."""

    def __init__(self, coop, g, srcs, threads=512, verify_host=None):
        import torch
        self.coop, self.g, self.srcs, self.threads = coop, g, list(srcs), threads
        info = coop.device_query(g.col_idx.device.index or 0, threads)
        self.N = info["max_coresident"] - 1                  # workers; +1 scheduler CTA
        out = torch.empty(g.num_vertices, dtype=torch.int32, device=g.col_idx.device)
        deg = g.degrees()
        self.m = {}
        for s in self.srcs:                                  # Graph500 edge count per source (untimed)
            coop.bfs(g, s, out, threads_per_wg=threads, flags=coop.FLAG_DIROPT)
            self.m[s] = int(deg[out >= 0].sum().item()) // 2
        self.verify_host = verify_host
        self.checks = []

    def loop(self, loop_s, **kw):
        coop = self.coop
        lv, runs, t_end, st = coop.bfs_loop(self.g, self.srcs, loop_s, threads_per_wg=self.threads,
                                            flags=coop.FLAG_DIROPT, event_cap=4096, **kw)
        last = self.srcs[(runs - 1) % len(self.srcs)]
        if self.verify_host is not None:
            self.checks.append((last, lv.cpu().numpy()))
        edges = sum(self.m[self.srcs[r % len(self.srcs)]] for r in range(runs))
        T = float(t_end[-1]) if len(t_end) else 0.0
        return {"runs": runs, "loop_s": T, "ms_per_bfs": 1e3 * T / max(1, runs),
                "gteps": edges / T / 1e9 if T else None}, st

    def standalone(self, loop_s, barriers=("query",)):
        """The loop with the scheduler armed and no task, per resizing-barrier implementation
        (the query barrier runs the scheduler-armed kernel with mid-interval offer_kill and
        hand-back, the naive barrier the general one), so a cell's slowdown compares like with like."""
        coop = self.coop
        self.base = getattr(self, "base", {})
        for b in barriers:
            r, st = self.loop(loop_s, max_wgs=self.N, policy=coop.POLICY_SCHEDULER,
                              barrier_mode=coop.BARRIER_QUERY if b == "query" else coop.BARRIER_NAIVE)
            self.base[b] = r
        return self.base[barriers[0]]

    def cell(self, preset, q, barrier, loop_s):
        coop = self.coop
        P_ms, E_ms = PRESETS_MS[preset]
        blocks = 10 * self.N
        block_ns = int(E_ms * 1e6 / 10)
        r, st = self.loop(loop_s, max_wgs=self.N, policy=coop.POLICY_SCHEDULER,
                          barrier_mode=coop.BARRIER_QUERY if barrier == "query" else coop.BARRIER_NAIVE,
                          task_wgs=q, task_blocks=blocks, task_block_ns=block_ns,
                          task_period_ns=int(P_ms * 1e6), task_first_ns=0)
        ev = st.task_events
        kill = [(e["t_first_start"] - e["t_arrive"]) / 1e3 for e in ev if e["t_first_start"]]
        gat = [(e["t_last_surrender"] - e["t_arrive"]) / 1e3 for e in ev if e["t_last_surrender"]]
        exe = [(e["t_end"] - e["t_first_start"]) / 1e6 for e in ev if e["t_end"] and e["t_first_start"]]
        arr = [e["t_arrive"] for e in ev if e["t_arrive"]]
        per = [(b - a) / 1e6 for a, b in zip(arr, arr[1:])]
        r.update({"preset": preset, "P_ms": P_ms, "E_ms": E_ms, "Q": q, "barrier": barrier,
                  "slowdown": r["ms_per_bfs"] / self.base[barrier]["ms_per_bfs"],
                  "kill_latency_us_p50": pct(kill, 0.5), "kill_latency_us_p99": pct(kill, 0.99),
                  "gather_us_p50": pct(gat, 0.5), "gather_us_p99": pct(gat, 0.99),
                  "task_exec_ms_mean": statistics.mean(exe) if exe else None,
                  "achieved_period_ms": statistics.mean(per) if per else None,
                  "tasks_completed": st.tasks_completed, "kills": st.kills, "forks": st.forks,
                  "mid_kills": st.mid_kills})
        return r

    def verify(self):
        """Last run of every loop == the oracle (C textbook BFS), run on the host cores."""
        import numpy as np
        from oracle import textbook as tb
        gh = self.verify_host
        ro = gh.row_offsets.numpy().astype(np.int64)
        col = gh.col_idx.numpy()
        srcs = sorted({s for s, _ in self.checks})
        with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
            ref = dict(zip(srcs, ex.map(lambda s: tb.bfs_arrays(gh.num_vertices, ro, col, s), srcs)))
        bad = [int(s) for s, lv in self.checks if not np.array_equal(lv, ref[s])]
        return {"verified": not bad, "loops_checked": len(self.checks), "mismatched_sources": bad}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--loop-s", type=float, default=10.0)
    ap.add_argument("--cells", default="all", choices=["all", "bench"])
    ap.add_argument("--threads", type=int, default=512)
    args = ap.parse_args()
    import torch
    import graphgen as gg
    from paper_1707_01989_b200 import coop
    coop.load()
    g = gg.rmat(args.scale, seed=1, device="cuda", chunk=1 << 26)
    srcs = gg.sample_sources(g, 64, seed=2)
    mt = MultitaskRunner(coop, g, srcs, args.threads, verify_host=g.to("cpu"))
    N = mt.N
    mt.standalone(args.loop_s, barriers=("query", "naive") if args.cells == "all" else ("query",))
    print(json.dumps({"standalone": mt.base, "N": N, "graph": f"rmat{args.scale}",
                      "gpu": torch.cuda.get_device_name()}), flush=True)
    qs = [1, N // 4, N // 2, N - 1]
    cells = ([(p, q, b) for p in PRESETS_MS for q in qs for b in ("query", "naive")] if args.cells == "all"
             else [(p, N // 4, "query") for p in PRESETS_MS])
    for p, q, b in cells:
        print(json.dumps(mt.cell(p, q, b, args.loop_s)), flush=True)
    print(json.dumps({"parity": mt.verify()}), flush=True)


if __name__ == "__main__":
    main()
