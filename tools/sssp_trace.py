"""Per-episode timeline of the cooperative near-far SSSP on the 2048^2 grid (GPU box; a
-DCOOP_LTRACE=1 build, prebuilt at build_variants/libcoop_ltrace.so).  The trace keeps the
first 63 episodes; prints the median over them of: expand (first start -> last end),
end imbalance (median -> last end), arrival, serial section, publish, release seen, and
the whole episode (release -> next release).
    python tools/sssp_trace.py [delta]
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
from paper_1707_01989_b200 import coop  # noqa: E402

lib_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build_variants",
                        "libcoop_ltrace.so")
coop.load(lib_path)
lib = ctypes.CDLL(lib_path)
lib.coop_debug_ltrace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
delta = int(sys.argv[1]) if len(sys.argv) > 1 else 16000
g = gg.with_weights(gg.grid(2048, 2048, device="cuda"), seed=1)
g.max_weight = 1000
out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
buf = np.zeros((64, 1184, 12), dtype=np.uint64)
for thr, wgs in ((512, 148), (256, 296)):
    lib.coop_debug_ltrace(None, 0)
    _, st = coop.sssp(g, 0, out, threads_per_wg=thr, max_wgs=wgs, sssp_delta=delta, level_cap=64)
    torch.cuda.synchronize()
    assert lib.coop_debug_ltrace(buf.ctypes.data, buf.size) == 0
    n = wgs
    ph = {k: [] for k in ("expand", "imbalance", "arrival", "serial", "publish", "seen", "episode")}
    for L in range(1, 62):
        t = buf[L, :n].astype(np.int64)
        t1 = buf[L + 1, :n].astype(np.int64)
        if not (t[:, 0] > 0).all() or not (t1[:, 0] > 0).all():
            break
        s0, e50, emax = t[:, 0].min(), np.median(t[:, 1]), t[:, 1].max()
        arr = t[:, 8].max()
        pre = t[:, 9][t[:, 9] > 0].max() if (t[:, 9] > 0).any() else arr
        pub = t[:, 10][t[:, 10] > 0].max() if (t[:, 10] > 0).any() else pre
        seen = t[:, 11][t[:, 11] > 0].max() if (t[:, 11] > 0).any() else pub
        ph["expand"].append(emax - s0); ph["imbalance"].append(emax - e50); ph["arrival"].append(arr - emax)
        ph["serial"].append(pre - arr); ph["publish"].append(pub - pre); ph["seen"].append(seen - pub)
        ph["episode"].append(t1[:, 0].min() - s0)
    print(json.dumps({"threads": thr, "wgs": wgs, "delta": delta, "ms": st.kernel_ns / 1e6, "episodes": st.levels,
                      "median_us": {k: round(float(np.median(v)) / 1e3, 2) for k, v in ph.items() if v}}), flush=True)
