import torch, graphgen as gg
from paper_1707_01989_b200 import coop
g = gg.rmat(24, seed=1, device="cuda", chunk=1 << 26)
deg = g.degrees()
iso = int((deg == 0).nonzero()[0].item())
out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
l2 = torch.empty(1 << 26, dtype=torch.int32, device="cuda")
for flags in (coop.FLAG_DIROPT, 0):
    ks = []
    for rep in range(5):
        l2.fill_(rep)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); _, st = coop.bfs(g, iso, out, threads_per_wg=512, flags=flags); e1.record(); torch.cuda.synchronize()
        ks.append((st.kernel_ns / 1e3, e0.elapsed_time(e1) * 1e3))
    print("flags", flags, "isolated-source BFS: kernel_us (globaltimer), event_us:", ks[1:])
