"""Host-side cost of one coop.bfs call (tiny graph): wall time per call vs kernel time."""
import time
import torch
import graphgen as gg
from paper_1707_01989_b200 import coop

g = gg.grid(8, 8).to("cuda")
out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
for _ in range(20):
    coop.bfs(g, 0, out)
torch.cuda.synchronize()
for flags in (0, coop.FLAG_DIROPT):
    n = 200
    t = time.perf_counter()
    ks = 0
    for _ in range(n):
        _, st = coop.bfs(g, 0, out, flags=flags)
        ks += st.kernel_ns
    dt = (time.perf_counter() - t) / n
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        coop.bfs(g, 0, out, flags=flags)
    e1.record()
    torch.cuda.synchronize()
    print(f"flags {flags}: wall {dt * 1e6:.1f} us/call, event {e0.elapsed_time(e1) * 1e3 / n:.1f} us/call, "
          f"kernel (globaltimer) {ks / n / 1e3:.1f} us")
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    coop.bfs(g, 0, out)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
