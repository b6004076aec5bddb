#!/usr/bin/env python
"""bench.py -- cooperative BFS on B200 (BASELINE.json metric: GTEPS; configs[2]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--scale S] [--quick]

A step = one cooperative BFS (the whole hot path of SURVEY §8(a): persistent
launch, init, per-level expand/claim/compact, resizing barriers, termination)
from one source of RMAT-24 (Graph500 parameters, seed 1), inputs
resident in HBM.  Sources are distinct degree>0 vertices (seed 2).  The job is
the K traversals, issued as asynchronous calls (coop_bfs_launch) on one stream
with two in flight; time = CUDA events around the whole sequence on the
launching stream (--serial: one blocking call per step, each bracketed by
events, L2 flushed before each).  The CSR (2.2 GB) is larger than the 126 MB
L2.  value = GTEPS (Graph500 convention: undirected edges of the reached
component / time); every timed output is compared with the oracle.  Extra objects report the multitasked run (periodic
competing task), the non-cooperative persistent baseline, ns per barrier vs the
L2 atomic round trip, and SSSP on the 2048x2048 grid (configs[1]).

--impl reference times the oracle (oracle/textbook.c, 1 host core) on the same
workload: the base contract's reference arm for this tier.
Under torchrun (N>1): the 1-D vertex-partitioned BFS (configs[4]),
weak scaling with 2^24 vertices per GPU, frontier exchanged inside the kernel
over NVLink peer memory (--exchange nccl: per-level ncclAllGather); time = max
over ranks, rank 0 prints.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BFS/SSSP GTEPS at 1/2/4/8 B200 (alone vs multitasked); barrier ns; kill latency"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for n, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def alg_bytes_bfs(st, V):
    """Algorithmic HBM bytes of one cooperative BFS launch:
    4 B per column index examined (top-down scans + bottom-up checks), 20 B per
    reached vertex (frontier entry read 4 + row offsets 8 + level write 4 +
    append 4), the level init 4V + V/8 bitmap, and per bottom-up level the
    sequential row-offset read 4V plus the visited and frontier bitmaps 3V/8."""
    return (4 * st.edges_scanned + 20 * st.reached + 4 * V + V // 8
            + st.bottom_up_levels * (4 * V + 3 * V // 8))


def make_graph(scale, device):
    import graphgen as gg
    t = time.time()
    g = gg.rmat(scale, seed=1, device=device, chunk=1 << 26)
    return g, time.time() - t


def oracle_gteps(g_host, sources, budget_s, deg):
    """Time the oracle (C textbook BFS, 1 core) on as many sources as fit the budget."""
    import numpy as np
    from oracle import textbook as tb
    ro = g_host.row_offsets.numpy().astype(np.int64)
    col = g_host.col_idx.numpy()
    V = g_host.num_vertices
    edges = 0
    secs = 0.0
    n = 0
    for s in sources:
        t = time.perf_counter()
        lv = tb.bfs_arrays(V, ro, col, s)
        secs += time.perf_counter() - t
        edges += int(deg[lv >= 0].sum()) // 2
        n += 1
        if secs >= budget_s:
            break
    return edges / secs / 1e9, n, secs


def verify_levels(g_host, results):
    """Parity at the benchmarked size: every level array the GPU produced
    for a timed source is compared element by element with the oracle (C textbook
    BFS) on the same graph; the oracle runs are spread over the host's cores (ctypes
    releases the GIL).  Returns {"verified": bool, "sources_checked": n, ...}."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    from oracle import textbook as tb
    ro = g_host.row_offsets.numpy().astype(np.int64)
    col = g_host.col_idx.numpy()
    V = g_host.num_vertices
    srcs = sorted({s for s, _ in results})
    t = time.perf_counter()
    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        ref = dict(zip(srcs, ex.map(lambda s: tb.bfs_arrays(V, ro, col, s), srcs)))
    bad = [int(s) for s, lv in results if not np.array_equal(lv.cpu().numpy(), ref[s])]
    return {"verified": not bad, "outputs_checked": len(results), "sources_checked": len(srcs),
            "mismatched_sources": bad[:8], "oracle_s": round(time.perf_counter() - t, 1),
            "how": "levels of every timed traversal == oracle/textbook.c, element by element"}


def run_reference(args, ws, rank):
    if rank != 0:
        return
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    g, _ = make_graph(args.scale, dev)
    import graphgen as gg
    srcs = gg.sample_sources(g, 64, seed=2)
    gh = g.to("cpu")
    deg = gh.degrees().numpy()
    del g
    import numpy as np
    from oracle import textbook as tb
    ro = gh.row_offsets.numpy().astype(np.int64)
    col = gh.col_idx.numpy()
    V = gh.num_vertices
    times, edges = [], []
    for i in range(args.warmup + args.steps):
        s = srcs[i % len(srcs)]
        t = time.perf_counter()
        lv = tb.bfs_arrays(V, ro, col, s)
        dt = time.perf_counter() - t
        if i >= args.warmup:
            times.append(dt)
            edges.append(int(deg[lv >= 0].sum()) // 2)
    val = sum(edges) / sum(times) / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GTEPS", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (RMAT, Graph500 parameters, seeded)",
            "config": {"workload": f"BFS RMAT-{args.scale} (configs[2]) from {args.steps} sources",
                       "scale": args.scale, "edgefactor": 16, "vertices": V, "directed_edges": gh.num_edges},
            "cpu_baseline": {"value": val, "unit": "GTEPS", "cores": 1, "kind": "oracle",
                             "sample": f"{args.steps} full single-source BFS runs of oracle/textbook.c"},
            "e2e": {"value": val, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, ws, rank, local):
    import numpy as np
    import torch
    import graphgen as gg
    from paper_1707_01989_b200 import coop

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    coop.load()
    info = coop.device_query(local, args.threads)
    g, gen_s = make_graph(args.scale, dev)
    V, E = g.num_vertices, g.num_edges
    deg = g.degrees()
    srcs = gg.sample_sources(g, 64, seed=2)
    # graph layout for BFS (once per graph, untimed like the graph generation): hub-first
    # neighbour order, probe records, degree-zero bitmap -- built by libcoop kernels
    # (coop_csr_hub_first / coop_csr_probe / coop_csr_isolated)
    torch.cuda.synchronize(dev)
    t_lay = time.time()
    coop._bfs_csr(g)
    torch.cuda.synchronize(dev)
    layout_s = time.time() - t_lay
    out = torch.empty(V, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    n_steps = args.warmup + args.steps
    checked = []

    def one(i, **kw):
        s = srcs[(i + rank * 7) % len(srcs)]
        flush.fill_(i & 0xFF)                                # L2 flush (untimed)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(stream)                                    # materialise the cudaEvent handles;
        k1.record(stream)                                    # libcoop re-records them around the kernel
        e0.record(stream)
        _, st = coop.bfs(g, s, out, threads_per_wg=args.threads, ev_kernel_start=k0, ev_kernel_end=k1,
                         event_cap=kw.pop("event_cap", 0), **kw)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if rank == 0 and ws == 1 and not args.no_verify:
            checked.append((s, out.clone()))                # untimed (device copy): verified below
        return e0.elapsed_time(e1), k0.elapsed_time(k1), st

    # ---- main: standalone cooperative BFS (NeverResize).  The job is the K traversals: calls
    # are issued back to back on one stream with two in flight (workspaces 0/1), so the host
    # preparation of call i+1 overlaps the kernel of call i; time = CUDA events around the
    # whole sequence on the launching stream.  No L2 flush inside the sequence: the CSR
    # (2.2 GB) and the level arrays are larger than L2.  Per-call kernel events give the
    # roofline.  (--serial: one blocking call per step, L2 flushed before each.)
    flags = 0 if args.topdown else coop.FLAG_DIROPT
    outs = [torch.empty(V, dtype=torch.int32, device=dev) for _ in range(max(args.steps, args.warmup))]

    def pipelined(first, count):
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(count)]
        for k0, k1 in kev:                                   # materialise the handles (re-recorded by libcoop)
            k0.record(stream)
            k1.record(stream)
        flush.fill_(first & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        inflight, st_all = [], []
        for j in range(count):
            s = srcs[(first + j + rank * 7) % len(srcs)]
            inflight.append((s, j, coop.BfsCall(g, s, outs[j], threads_per_wg=args.threads, flags=flags,
                                                 workspace=j % 2, ev_kernel_start=kev[j][0],
                                                 ev_kernel_end=kev[j][1])))
            if len(inflight) == 2:
                s0, j0, c0 = inflight.pop(0)
                st_all.append((s0, j0, c0.wait()))
        e1.record(stream)
        for s0, j0, c0 in inflight:
            st_all.append((s0, j0, c0.wait()))
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1), [k0.elapsed_time(k1) for k0, k1 in kev], st_all

    if args.serial:
        for i in range(args.warmup):
            one(i, flags=flags)
    else:
        pipelined(0, args.warmup)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    times, ktimes, stats = [], [], []
    with ClockSampler(local) as clk:
        if args.serial:
            for i in range(args.warmup, n_steps):
                t, kt, st = one(i, flags=flags)
                times.append(t)
                ktimes.append(kt)
                stats.append(st)
                # Graph500 edge count of this traversal, from the result (untimed)
                st.teps_edges = int(deg[out >= 0].sum().item()) // 2
        else:
            tot, ktimes, st_all = pipelined(args.warmup, args.steps)
            times = [tot / args.steps] * args.steps
            for s0, j0, st in st_all:
                st.teps_edges = int(deg[outs[j0] >= 0].sum().item()) // 2
                stats.append(st)
                if rank == 0 and ws == 1 and not args.no_verify:
                    checked.append((s0, outs[j0].clone()))
    torch.cuda.synchronize(dev)
    tot_ms = sum(times)
    if ws > 1:
        t = torch.tensor([tot_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_ms = float(t.item())
        ed = torch.tensor([float(sum(s.teps_edges for s in stats))], device=dev)
        torch.distributed.all_reduce(ed)
        all_edges = float(ed.item())
    else:
        all_edges = float(sum(s.teps_edges for s in stats))
    gteps = all_edges / (tot_ms * 1e-3) / 1e9
    peak, peak_src = _peaks()
    alg_bytes = [alg_bytes_bfs(st, V) for st in stats]
    achieved = sum(alg_bytes) / (sum(ktimes) * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            key = "bfs_rmat%d_%s" % (args.scale, "topdown" if args.topdown else "diropt")
            traffic = json.load(open(prof)).get(key, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    extras = {}
    if rank == 0 and not args.quick:
        extras = run_extras(args, g, srcs, out, flush, stream, dev, info, times, flags, checked)

    # ---- end to end through the C ABI with HOST buffers (H2D graph + D2H levels inside)
    e2e = None
    if rank == 0:
        ro_h = g.row_offsets.to(torch.int32).cpu().pin_memory()
        col_h = g.col_idx.cpu().pin_memory()
        lv_h = torch.empty(V, dtype=torch.int32).pin_memory()
        et, ee = [], []
        deg_h = deg.cpu()
        for i in range(1 + 3):
            s = srcs[i]
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            coop.bfs_host(ro_h, col_h, s, lv_h, threads_per_wg=args.threads, flags=flags)
            dt = time.perf_counter() - t0
            if i >= 1:
                et.append(dt)
                ee.append(int(deg_h[lv_h >= 0].sum()) // 2)
        e2e = {"value": sum(ee) / sum(et) / 1e9, "unit": "GTEPS",
               "h2d_bytes_per_step": int(ro_h.numel() * 4 + col_h.numel() * 4),
               "d2h_bytes_per_step": int(V * 4), "steps": len(et)}
        del ro_h, col_h
    # ---- parity of every timed output (and the multitasked runs) against the oracle
    verify = None
    if rank == 0 and ws == 1 and not args.no_verify:
        verify = verify_levels(g.to("cpu"), checked)
        checked.clear()
    # ---- CPU oracle baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        gh = g.to("cpu")
        dh = gh.degrees().numpy()
        v, n, secs = oracle_gteps(gh, srcs, args.cpu_budget, dh)
        cpu = {"value": v, "unit": "GTEPS", "cores": 1, "kind": "oracle",
               "sample": f"{n} single-source BFS runs of oracle/textbook.c on the same RMAT-{args.scale} "
                         f"({secs:.1f} s of CPU work)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": gteps, "unit": "GTEPS", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (RMAT, Graph500 parameters a,b,c=.57,.19,.19, edgefactor 16, seed 1, relabelled)",
            "config": {"workload": f"BFS RMAT-{args.scale} (configs[2]), standalone cooperative, NeverResize, "
                                   + ("top-down" if args.topdown else "direction-optimising (top-down + bottom-up levels)"),
                       "scale": args.scale, "vertices": V, "directed_edges": E, "sources": args.steps,
                       "wgs": info["max_coresident"], "threads_per_wg": args.threads,
                       "l2": ("flushed (256 MB write) before every step; CSR 2.2 GB > L2" if args.serial else
                              "inputs larger than L2 (CSR 2.2 GB + 67 MB levels); no flush inside the sequence"),
                       "calls": "one blocking call per step" if args.serial else
                                "pipelined: 2 asynchronous calls in flight on one stream (coop_bfs_launch)",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU",
                       "graph_gen_s": round(gen_s, 2),
                       "layout": ("hub-first neighbour order + probe records + degree-zero bitmap"
                                  if coop.USE_HUB_FIRST else
                                  "generator order + probe records" if coop.USE_PROBE else "generator order"),
                       "layout_s": round(layout_s, 3)},
            "kernel_ms_per_step": sum(ktimes) / len(ktimes),
            "levels": stats[-1].levels, "bottom_up_levels": stats[-1].bottom_up_levels,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "coop_kernel<BfsApp<uint32_t>,%d>" % args.threads,
                         "alg_bytes_per_launch": sum(alg_bytes) / len(alg_bytes)},
            "cpu_baseline": cpu,
            "parity": verify,
            "e2e": e2e,
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            **extras,
        }
        print(json.dumps(line), flush=True)
        if verify is not None and not verify["verified"]:
            sys.exit(f"bench: GPU levels differ from the oracle for sources {verify['mismatched_sources']}")
    if ws > 1:
        torch.distributed.destroy_process_group()


def run_extras(args, g, srcs, out, flush, stream, dev, info, base_times, flags, checked):
    import torch
    import graphgen as gg
    from paper_1707_01989_b200 import coop
    ex = {}
    N = info["max_coresident"]

    deg = g.degrees()                   # Graph500 edge counts of the multitasked runs (R18)

    def timed(fn):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1), r

    k = min(args.steps, 8)
    # C3 as SURVEY 8(d) states it: the 64 sources, one call each (L2 flushed, CUDA events around the
    # call), GTEPS aggregated by harmonic mean (Graph500); every 8th output is checked by the oracle
    per, perk = [], []
    for i, s64 in enumerate(srcs[:64]):
        t, (_, st) = timed(lambda: coop.bfs(g, s64, out, threads_per_wg=args.threads, flags=flags))
        e = int(deg[out >= 0].sum().item()) // 2
        per.append(e / (t * 1e-3) / 1e9)
        perk.append(e / (st.kernel_ns * 1e-9) / 1e9)
        if not args.no_verify and i % 8 == 0:
            checked.append((s64, out.clone()))
    hmean = lambda xs: len(xs) / sum(1.0 / x for x in xs)
    ex["c3_64_sources"] = {"sources": len(per), "gteps_harmonic_mean": hmean(per),
                           "gteps_harmonic_mean_kernel": hmean(perk), "gteps_min": min(per), "gteps_max": max(per),
                           "timing": "one call per source (not pipelined), CUDA events around the call, L2 flushed; "
                                     "_kernel: the kernel's own %globaltimer span"}
    # T2 analogue: the cooperative kernel with no competing task against the
    # separately compiled non-cooperative persistent kernel (kCoop = false: plain barrier,
    # static split, no scheduler/pool/mailbox code), all at the same N worker CTAs.  Two
    # cooperative arms: the scheduler never resizes (NEVER) and the scheduler armed with no
    # task (SCHEDULER: scheduler CTA running, chunk claims + demand reads in every interval,
    # the kernel "still interacts with the scheduler").  Ratios are geometric
    # means over sources of per-source medians (the paper's aggregation).
    n_w = N - 1
    arms = {"noncoop": dict(barrier_mode=coop.BARRIER_PLAIN),
            "coop_never": dict(),
            "coop_scheduler_armed": dict(policy=coop.POLICY_SCHEDULER)}
    per = {a: [] for a in arms}
    n_src = max(8, k)
    for i in range(n_src):
        samples = {a: [] for a in arms}
        for rep in range(3):
            for a, kw in arms.items():
                t, _ = timed(lambda: coop.bfs(g, srcs[i], out, threads_per_wg=args.threads, max_wgs=n_w,
                                              flags=flags, **kw))
                samples[a].append(t)
        for a in arms:
            per[a].append(statistics.median(samples[a]))

    def geo(xs):
        import math
        return math.exp(sum(math.log(x) for x in xs) / len(xs))
    ex["noncoop_baseline"] = {
        "workers": n_w, "sources": n_src, "ms_median": {a: statistics.median(v) for a, v in per.items()},
        "slowdown_never_vs_noncoop": geo([c / b for c, b in zip(per["coop_never"], per["noncoop"])]),
        "slowdown_armed_vs_noncoop": geo([c / b for c, b in zip(per["coop_scheduler_armed"], per["noncoop"])]),
        "aggregation": "geomean over sources of per-source medians of 3 interleaved runs"}
    t_coop = per["coop_never"]
    # the north_star path alone: pure top-down BFS (expand / claim / compact every level, no
    # bottom-up levels) with its own roofline (same algorithmic-bytes formula)
    td_t, td_b, td_e = [], [], 0
    for i in range(k):
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.fill_(2)
        k0.record(stream)
        k1.record(stream)
        _, st = coop.bfs(g, srcs[i], out, threads_per_wg=args.threads, ev_kernel_start=k0, ev_kernel_end=k1)
        torch.cuda.synchronize(dev)
        td_t.append(k0.elapsed_time(k1))
        td_b.append(alg_bytes_bfs(st, g.num_vertices))
        td_e += int(g.degrees()[out >= 0].sum().item()) // 2
        if not args.no_verify:
            checked.append((srcs[i], out.clone()))
    peak, _ = _peaks()
    ach = sum(td_b) / (sum(td_t) * 1e-3) / 1e9
    ex["bfs_topdown"] = {"kernel_ms_mean": statistics.mean(td_t), "gteps": td_e / (sum(td_t) * 1e-3) / 1e9,
                         "sources": k, "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                                                    "frac": ach / peak,
                                                    "alg_bytes_per_launch": sum(td_b) / len(td_b)},
                         "note": "top-down only (FLAG_DIROPT off): the north_star expand/claim/compact path"}
    # multitasked: scheduler CTA posts a task every P with Q = N/4 WGs (scaled light preset)
    mt = {}
    for name, (P_us, E_us) in {"stress": (200, 20)}.items():
        q = max(1, (N - 1) // 4)
        blocks = 4 * q
        block_ns = int(E_us * 1000 * (N - 1) / blocks)
        tt, lat, gat, tasks, tedges, mk, hb, rp = [], [], [], 0, 0, 0, 0, 0
        for i in range(k + 1):
            t, (_, st) = timed(lambda: coop.bfs(g, srcs[i], out, threads_per_wg=args.threads, flags=flags,
                                                policy=coop.POLICY_SCHEDULER, task_wgs=q, task_blocks=blocks,
                                                task_block_ns=block_ns, task_period_ns=P_us * 1000,
                                                task_first_ns=0, event_cap=4096))
            if i:
                tt.append(t)
                tasks += st.tasks_completed
                mk += st.mid_kills
                hb += st.handbacks
                rp += st.replays
                tedges += int(deg[out >= 0].sum().item()) // 2     # Graph500 count (R18), untimed
                if not args.no_verify:
                    checked.append((srcs[i], out.clone()))          # multitasked levels: same oracle
                for e in st.task_events:
                    if e["t_first_start"]:
                        lat.append((e["t_first_start"] - e["t_arrive"]) / 1e3)
                    if e["t_last_surrender"]:
                        gat.append((e["t_last_surrender"] - e["t_arrive"]) / 1e3)
        # standalone reference with the scheduler CTA present (N-1 workers)
        def pct(v, p):
            v = sorted(v)
            return v[min(len(v) - 1, int(p * len(v)))] if v else None
        mt[name] = {"period_us": P_us, "work_us_at_full": E_us, "task_wgs": q,
                    "ms_per_bfs": statistics.median(tt),
                    "slowdown_vs_standalone": statistics.median(tt) / statistics.median(t_coop),
                    "kill_latency_us_p50": pct(lat, 0.5), "kill_latency_us_p99": pct(lat, 0.99),
                    "gather_us_p50": pct(gat, 0.5), "gather_us_p99": pct(gat, 0.99),
                    "tasks_completed": tasks, "gteps": tedges / (sum(tt) * 1e-3) / 1e9,
                    "mid_kills": mk, "handbacks": hb, "replays": rp}
    ex["multitask"] = mt
    # the paper's presets at Q = N/4 (query barrier), BFS looped over sources inside ONE
    # launch for >= 10 s per cell; the full preset x Q x barrier grid is
    # tools/multitask_paper.py (profiles/)
    if not args.no_paper_multitask:
        import importlib.util
        spec = importlib.util.spec_from_file_location("multitask_paper",
                                                      os.path.join(ROOT, "tools", "multitask_paper.py"))
        mp = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mp)
        runner = mp.MultitaskRunner(coop, g, srcs, args.threads,
                                    verify_host=None if args.no_verify else g.to("cpu"))
        base = runner.standalone(args.loop_s)
        cells = [runner.cell(p, runner.N // 4, "query", args.loop_s) for p in mp.PRESETS_MS]
        ex["multitask_paper"] = {"standalone_loop": base, "workers": runner.N, "cells": cells,
                                 "parity": runner.verify() if not args.no_verify else None,
                                 "note": "BFS looped over 64 sources inside one launch, loop_s each; task = "
                                         "E ms of work on all N workgroups every P ms, Q = N/4 demanded"}
    # barrier ns vs L2 atomic RTT (configs[3] points)
    rtt = coop.l2_atomic_rtt(50000)             # median over 8 SMs of a relaxed 64-bit atomic chain
    lat = coop.l2_latency_profile(20000)
    bar = {}
    for n in (148, 592, 1184):
        r = coop.barrier_bench(n, 200000, threads=128, plain=True)
        r2 = coop.barrier_bench(n, 200000, threads=128, resize_prob=1 / 64, seed=3)
        bar[str(n)] = {"plain_ns": r["ns_per_barrier"], "resizing_p1_64_ns": r2["ns_per_barrier"],
                       "kills": r2["kills"], "forks": r2["forks"]}
    # the round trip is bimodal: SMs on the die of the word's L2 slice see ~160 ns, the others
    # ~370 ns, so a median over 8 SMs lands on either; the barrier words sit on one die and every
    # barrier has CTAs on both, so both round trips are reported beside the median
    a64 = lat.get("atom_relaxed_u64", {})
    rtt_near, rtt_far = a64.get("min", rtt), a64.get("max", rtt)
    for n in bar:
        bar[n]["plain_over_rtt"] = bar[n]["plain_ns"] / rtt
        bar[n]["plain_over_rtt_near_die"] = bar[n]["plain_ns"] / rtt_near
        bar[n]["plain_over_rtt_far_die"] = bar[n]["plain_ns"] / rtt_far
    ex["barrier"] = {"l2_atomic_rtt_ns": rtt, "rtt_def": "dependent atom.relaxed.gpu.add.u64 chain, one thread, "
                     "median over 8 SMs on both dies", "rtt_near_die_ns": rtt_near, "rtt_far_die_ns": rtt_far,
                     "l2_latency_profile_ns": lat, "per_ctas": bar}
    # SSSP on the 2048x2048 grid (configs[1])
    gw = gg.with_weights(gg.grid(2048, 2048, device=dev), seed=1)
    gw.max_weight = 1000
    dout = torch.empty(gw.num_vertices, dtype=torch.int32, device=dev)
    m_und = gw.num_edges // 2
    ss = {}
    # plain worklist Bellman-Ford (delta 0) and the near-far pile (delta = band width);
    # distances are identical, only the work and the number of barrier episodes differ
    # near-far band width 16000 (x16 the largest weight): profiles/r02_sssp_sweep.log
    for name, delta, thr, n in (("bellman_ford", 0, 256, 148), ("near_far", 16000, 512, 148)):
        ts = []
        for i in range(3):
            t, (_, st) = timed(lambda: coop.sssp(gw, 0, dout, threads_per_wg=thr, max_wgs=n, sssp_delta=delta))
            if i:
                ts.append(t)
        ms = statistics.median(ts)
        E_R = gw.num_edges                                  # every vertex is reached on the grid
        V_R = gw.num_vertices
        lb = 8 * E_R + 20 * V_R                             # each vertex expanded once
        est = 20 * st.frontier_total + 16 * st.edges_scanned   # entries x (4 id + 8 key + 8 offsets), edges x (4+4+8)
        peak, _ = _peaks()
        ss[name] = {"ms": ms, "gteps": m_und / (ms * 1e-3) / 1e9, "delta": delta, "threads_per_wg": thr, "wgs": n,
                    "episodes": st.episodes, "relaxed_edges": st.edges_scanned,
                    "us_per_episode": ms * 1e3 / max(1, st.episodes),
                    "work_efficiency": st.edges_scanned / E_R,
                    "hbm_frac_lower_bound_bytes": lb / (ms * 1e-3) / 1e9 / peak,
                    "hbm_frac_executed_bytes": est / (ms * 1e-3) / 1e9 / peak,
                    "bound": "barrier latency (episodes x us_per_episode), not HBM"}
        if not args.no_verify:
            dlast = dout.cpu().numpy().view("uint32").copy()
            ss[name]["_dist"] = dlast
    # same-run oracle: Dijkstra (oracle/textbook.c, 1 host core) on the same grid, and parity
    import numpy as np
    from oracle import textbook as tb
    gh = gw.to("cpu")
    ro = gh.row_offsets.numpy().astype(np.int64)
    col = gh.col_idx.numpy()
    wts = gh.weights.numpy().astype(np.uint32)
    t0 = time.perf_counter()
    ref = tb.dijkstra_arrays(gh.num_vertices, ro, col, wts, 0)
    dj = time.perf_counter() - t0
    for name in ss:
        d = ss[name].pop("_dist", None)
        ss[name]["verified"] = None if d is None else bool(np.array_equal(d, ref))
    ss["dijkstra_oracle"] = {"s": dj, "gteps": m_und / dj / 1e9, "cores": 1,
                             "kind": "oracle (binary-heap Dijkstra, oracle/textbook.c)"}
    ex["sssp_grid2048"] = ss
    # device API (include/coop_device.cuh): the paper's Fig. 4 kernel written literally on
    # resizing_global_barrier (thread-strided, CAS claims), same RMAT-24 sources, and Fig. 2
    # work stealing with offer_kill / request_fork at the loop head (§3.2)
    m_graph = float(g.num_edges) / 2
    f4 = []
    with coop.DevHandle(policy=coop.POLICY_NEVER) as h:
        for i in range(3):
            t, (lv, st) = timed(lambda: coop.fig4_bfs(h, g, srcs[i], out, threads_per_wg=256))
            f4.append(t)
    ex["fig4_device_api_bfs"] = {"ms": statistics.median(f4), "episodes": st["episodes"],
                                 "note": "Fig. 4 literally on the device API (2 resizing barriers/level, "
                                         "thread-strided frontier, CAS claims); levels identical"}
    ws_line = {}
    tree = dict(seed=3, depth=18, max_fanout=4, rounds=16)
    for name, kw in (("never", dict(policy=coop.POLICY_NEVER)),
                     ("random_kill_fork", dict(policy=coop.POLICY_RANDOM, kill_prob=0.02, fork_prob=0.02,
                                               max_fork=8, seed=5))):
        ts, res = [], None
        with coop.DevHandle(**kw) as h:
            for i in range(3):
                t, (r, st) = timed(lambda: coop.work_steal(h, **tree))
                ts.append(t)
                res = r if res is None else res
                assert (r["count"], r["total"]) == (res["count"], res["total"])   # schedule independent
        ms = statistics.median(ts)
        ws_line[name] = {"ms": ms, "tasks": res["count"], "mtasks_per_s": res["count"] / ms / 1e3,
                         "steals": r["steals"], "kills": st["kills"], "forks": st["forks"], "wgs": st["n_wgs"]}
    ws_line["tree"] = tree
    ex["work_stealing_device_api"] = ws_line
    del m_graph
    return ex


def run_partitioned(args, ws, rank, local):
    """N > 1: the 1-D vertex-partitioned cooperative BFS (configs[4]) with the
    frontier all-gather inside the kernel over NVLink peer memory.  Weak
    scaling: RMAT scale = --scale + log2(N) (2^24 vertices per GPU; N=8 is
    RMAT-27).  value = Graph500 edges of the traversal / max-over-ranks time."""
    import math
    import torch
    import torch.distributed as dist
    import graphgen as gg
    from paper_1707_01989_b200 import coop, partitioned as pt
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    coop.load()
    scale = args.scale + int(round(math.log2(ws)))
    t0 = time.time()
    part = gg.rmat_partition(scale, ws, rank, seed=1, device=dev, chunk=1 << 26)
    gen_s = time.time() - t0
    V = part.num_vertices
    vb, ve = part.v_begin, part.v_end
    indeg = torch.bincount(part.col_local.to(torch.int64), minlength=ve - vb)   # = degree (symmetric graph)
    pb = pt.PartitionedBFS(part, dev, exchange=args.exchange)
    if args.exchange == "nccl":
        pb.connect_nccl()                 # north_star's NCCL all-gather data plane
    else:
        pb.connect_ipc()                  # fused: in-kernel NVLink peer stores
    eg = torch.tensor([float(part.num_edges)], device=dev, dtype=torch.float64)
    dist.all_reduce(eg)
    pb.E_global = int(eg.item())
    # sources: seeded hash order over all vertices, keep the first with degree > 0 anywhere
    cand = torch.argsort(gg.splitmix64(torch.arange(V, dtype=torch.int64, device=dev) ^ 0x5EED2), stable=True)[:4096]
    own = (cand >= vb) & (cand < ve)
    ok = torch.zeros(cand.numel(), dtype=torch.int32, device=dev)
    ok[own] = (indeg[cand[own] - vb] > 0).to(torch.int32)
    dist.all_reduce(ok, op=dist.ReduceOp.MAX)
    srcs = cand[ok > 0][:64].tolist()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    times, edges = [], []
    n_steps = args.warmup + args.steps
    with ClockSampler(local) as clk:
        for i in range(n_steps):
            flush.fill_(i & 0xFF)
            dist.barrier()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            lv, st = pb.run(srcs[i % len(srcs)], threads_per_wg=args.threads,
                            flags=0 if args.topdown else coop.FLAG_DIROPT)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            if i >= args.warmup:
                times.append(e0.elapsed_time(e1))
                edges.append(int(indeg[lv[: ve - vb] >= 0].sum().item()))
    tot = torch.tensor([sum(times)], device=dev)
    dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ed = torch.tensor([float(sum(edges))], device=dev)
    dist.all_reduce(ed)
    tot_ms = float(tot.item())
    gteps = float(ed.item()) / 2 / (tot_ms * 1e-3) / 1e9
    if rank == 0:
        line = {"metric": METRIC, "value": gteps, "unit": "GTEPS", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "int32",
                "data": "synthetic (RMAT, Graph500 parameters, seed 1, relabelled), generated per rank",
                "config": {"workload": f"BFS RMAT-{scale} 1-D vertex-partitioned over {ws} GPUs (configs[4]), "
                                       + ("frontier all-gather by ncclAllGather per level (host relay)"
                                          if args.exchange == "nccl" else
                                          "frontier all-gather inside the cooperative kernel over NVLink peer memory"),
                           "exchange": args.exchange,
                           "scale": scale, "vertices": V, "parallelism": f"1-D partition x{ws}",
                           "l2": "flushed (256 MB write) before every step", "graph_gen_s": round(gen_s, 2)},
                "roofline": None, "cpu_baseline": None, "e2e": None, "gpu_launches": args.steps * ws,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    pb.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--threads", type=int, default=512)
    ap.add_argument("--topdown", action="store_true", help="main line without direction optimisation")
    ap.add_argument("--quick", action="store_true", help="skip the extra objects")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--serial", action="store_true",
                    help="main line: one blocking call per step with an L2 flush before each (default: pipelined)")
    ap.add_argument("--no-verify", action="store_true", help="skip the oracle comparison of the outputs")
    ap.add_argument("--no-paper-multitask", action="store_true", help="skip the 10 s paper-preset loops")
    ap.add_argument("--loop-s", type=float, default=10.0, help="seconds per multitask loop (>= 10: P:1045)")
    ap.add_argument("--exchange", default="nvlink", choices=["nvlink", "nccl"],
                    help="N > 1: frontier exchange of the partitioned BFS")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    if ws > 1:
        run_partitioned(args, ws, rank, local)
        return
    run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
