"""Measured analogue of Table 3: sharing the GPU between the
compute kernel and a periodic competing task by KERNEL-LEVEL preemption versus by
cooperative kernels.

Compute: BFS on RMAT-24 from a cycle of 64 sources, >= loop_s seconds.
Task: every P ms, E ms of work on all N workgroups (presets light (70,3),
medium (40,3), heavy (40,10) ms).

  kernel-level  -- one BFS launch at a time (non-cooperative persistent kernel);
                   when a task is due it is launched between two BFS launches on
                   the same stream (it preempts the compute at kernel granularity)
                   as N blocks of E ms, i.e. the whole GPU for E.  Overhead =
                   elapsed / standalone elapsed for the same BFS runs; the paper's
                   model predicts P / (P - D) with D = E (oracle/preemption.py).
  cooperative   -- coop_bfs_loop with the in-kernel scheduler posting the task
                   (Q = N/4 for light/medium, N/2 for heavy: Table 3's resources);
                   overhead = ms per BFS / standalone loop ms per BFS.

    python tools/preemption_compare.py [--loop-s 10]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PRESETS_MS = {"light": (70.0, 3.0), "medium": (40.0, 3.0), "heavy": (40.0, 10.0)}


def kernel_level(coop, g, srcs, out, N, loop_s, P_ms, E_ms, threads):
    """BFS launches back to back for loop_s; a task every P_ms inserted between launches."""
    import torch
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    t0 = time.perf_counter()
    next_task = t0 if P_ms else float("inf")
    runs = tasks = 0
    while time.perf_counter() - t0 < loop_s:
        now = time.perf_counter()
        if now >= next_task:
            coop.load().coop_spin_task(N, 128, int(E_ms * 1e6), stream.cuda_stream)
            tasks += 1
            next_task += P_ms / 1e3
        coop.bfs(g, srcs[runs % len(srcs)], out, threads_per_wg=threads, max_wgs=N, flags=coop.FLAG_DIROPT,
                 barrier_mode=coop.BARRIER_PLAIN)
        runs += 1
    e1.record(stream)
    torch.cuda.synchronize()
    return runs, tasks, e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--loop-s", type=float, default=10.0)
    ap.add_argument("--threads", type=int, default=512)
    args = ap.parse_args()
    import torch
    import graphgen as gg
    from oracle import preemption as pre
    from paper_1707_01989_b200 import coop
    spec = __import__("importlib.util").util.spec_from_file_location(
        "multitask_paper", os.path.join(ROOT, "tools", "multitask_paper.py"))
    mp = __import__("importlib.util").util.module_from_spec(spec)
    spec.loader.exec_module(mp)
    coop.load()
    g = gg.rmat(args.scale, seed=1, device="cuda", chunk=1 << 26)
    srcs = gg.sample_sources(g, 64, seed=2)
    out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
    runner = mp.MultitaskRunner(coop, g, srcs, args.threads)
    N = runner.N
    # kernel-level: standalone (no task), then each preset
    runs0, _, ms0 = kernel_level(coop, g, srcs, out, N, args.loop_s, 0, 0, args.threads)
    per0 = ms0 / runs0
    base = runner.standalone(args.loop_s)
    print(json.dumps({"standalone": {"kernel_level_ms_per_bfs": per0, "coop_loop_ms_per_bfs": base["ms_per_bfs"]},
                      "N": N}), flush=True)
    for name, (P_ms, E_ms) in PRESETS_MS.items():
        runs, tasks, ms = kernel_level(coop, g, srcs, out, N, args.loop_s, P_ms, E_ms, args.threads)
        kl = (ms / runs) / per0
        q = N // 2 if name == "heavy" else N // 4
        c = runner.cell(name, q, "query", args.loop_s)
        print(json.dumps({"preset": name, "P_ms": P_ms, "E_ms": E_ms,
                          "model_P_over_P_minus_D": pre.preemption_overhead(P_ms, E_ms),
                          "kernel_level_overhead": kl, "kernel_level_tasks": tasks,
                          "cooperative_overhead": c["slowdown"], "cooperative_Q": q,
                          "cooperative_tasks": c["tasks_completed"],
                          "cooperative_achieved_period_ms": c["achieved_period_ms"],
                          "cooperative_kill_latency_us_p50": c["kill_latency_us_p50"]}), flush=True)


if __name__ == "__main__":
    main()
