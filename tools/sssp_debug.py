import numpy as np, torch, ctypes
import graphgen as gg
from oracle import textbook as tb
from paper_1707_01989_b200 import coop
for (R, C) in ((48, 64), (37, 53), (100, 100)):
    g = gg.with_weights(gg.grid(R, C), seed=1)
    ref = tb.dijkstra(g, 0)
    gd = g.to("cuda")
    for thr, N in ((256, 0), (256, 4), (256, 1), (1024, 1)):
        d, st = coop.sssp(gd, 0, threads_per_wg=thr, max_wgs=N)
        a = d.cpu().numpy().view(np.uint32)
        bad = np.nonzero(a != ref)[0]
        print(R, C, thr, N, "bad", len(bad), [(int(v), int(a[v]), int(ref[v])) for v in bad[:4]], "rounds", st.levels)
