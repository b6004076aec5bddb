"""Per-level timeline of the cooperative BFS on RMAT-24 (GPU box).

Builds a -DCOOP_LTRACE=1 variant of the library (per-CTA %globaltimer stamps at
expand start / expand end / after barrier 1 / after barrier 2 of every level),
runs one BFS per source and prints, per level, in microseconds relative to the
previous level's release:
  start  : last CTA to begin the expand (after the barrier release + empty())
  end50 / end_max : median / last CTA to finish its expand
  rb1    : last CTA out of barrier 1;  rb2 : last CTA out of barrier 2
    python tools/level_trace.py [flags] [sources]
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
from paper_1707_01989_b200 import build, coop  # noqa: E402

lib_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build_variants", "libcoop_ltrace.so")
os.makedirs(os.path.dirname(lib_path), exist_ok=True)
if not (os.environ.get("LT_NOBUILD") and os.path.exists(lib_path)):   # prebuilt on the CPU side
    build.build(out=lib_path, defines=["COOP_LTRACE=1"])
coop.load(lib_path)
lib = ctypes.CDLL(lib_path)
lib.coop_debug_ltrace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]

flags = int(sys.argv[1]) if len(sys.argv) > 1 else coop.FLAG_DIROPT
# LT_POLICY=scheduler: the scheduler-armed arm (scheduler CTA, no task), N-1 workers
extra = {}
if os.environ.get("LT_POLICY") == "scheduler":
    extra = dict(policy=coop.POLICY_SCHEDULER)
if os.environ.get("LT_WORKERS"):
    extra["max_wgs"] = int(os.environ["LT_WORKERS"])
nsrc = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = gg.rmat(24, seed=1, device="cuda", chunk=1 << 26)
out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
buf = np.zeros((64, 1184, 12), dtype=np.uint64)
for s in gg.sample_sources(g, nsrc, seed=2):
    for rep in range(2):
        lib.coop_debug_ltrace(None, 0)
        _, st = coop.bfs(g, s, out, threads_per_wg=512, flags=flags, level_cap=64, **extra)
    torch.cuda.synchronize()
    rc = lib.coop_debug_ltrace(buf.ctypes.data, buf.size)
    assert rc == 0
    n_cta = st.n_wgs or 296
    rows = []
    prev = None
    for L in range(st.levels):
        t = buf[L, :n_cta].astype(np.int64)
        if prev is None:
            prev = int(t[:, 0].min())
        rel = (t - prev) / 1e3
        rows.append({"L": L, "size": st.level_sizes[L] if L < len(st.level_sizes) else None,
                     "start": round(float(rel[:, 0].max()), 1), "end50": round(float(np.median(rel[:, 1])), 1),
                     "end_max": round(float(rel[:, 1].max()), 1), "rb1": round(float(rel[:, 2].max()), 1),
                     "rb2": round(float(rel[:, 3].max()), 1) if (t[:, 3] > 0).any() else None,
                     # warp 0 of each CTA inside expand: after the bitmap recycle, after the
                     # heavy pass, after the claimed items, after the flush (median over CTAs)
                     "w0": [round(float(np.median(rel[:, k][t[:, k] > 0])), 1) if (t[:, k] > 0).any() else None
                            for k in (4, 5, 6, 7)],
                     # barrier #1 phases: last arrival (thread 0 after its atomic), the last
                     # arriver's serial section up to the publish, after it, the last waiter
                     # to see the release
                     "bar": {"arr_max": round(float(rel[:, 8].max()), 1) if (t[:, 8] > 0).any() else None,
                             "pre_pub": round(float(rel[:, 9][t[:, 9] > 0].max()), 1) if (t[:, 9] > 0).any() else None,
                             "pub": round(float(rel[:, 10][t[:, 10] > 0].max()), 1) if (t[:, 10] > 0).any() else None,
                             "seen_max": round(float(rel[:, 11][t[:, 11] > 0].max()), 1) if (t[:, 11] > 0).any() else None}})
        prev = int(t[:, 2].max())
    # kernel entry / init start / init done per CTA (slots of row 63), relative to the first entry
    e = buf[63, :n_cta, :3].astype(np.int64)
    t0 = int(e[:, 0][e[:, 0] > 0].min()) if (e[:, 0] > 0).any() else 0
    init = {"entry_max": round(float((e[:, 0].max() - t0) / 1e3), 1),
            "init_done_med": round(float((np.median(e[:, 2]) - t0) / 1e3), 1),
            "init_done_max": round(float((e[:, 2].max() - t0) / 1e3), 1),
            "L0_start_min": round(float((buf[0, :n_cta, 0].astype(np.int64).min() - t0) / 1e3), 1)} if t0 else None
    print(json.dumps({"src": s, "flags": flags, "kernel_us": st.kernel_ns / 1e3, "bu": st.bottom_up_levels,
                      "init": init, "levels": rows}), flush=True)
