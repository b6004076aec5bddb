import time, ctypes, torch
import graphgen as gg
from paper_1707_01989_b200 import coop
g = gg.grid(8, 8).to("cuda")
out = torch.empty(g.num_vertices, dtype=torch.int32, device="cuda")
for _ in range(20): coop.bfs(g, 0, out)
lib = coop.load()
c, keep = coop._device_csr(g, False)
n = 300
t = time.perf_counter()
for _ in range(n): o, k2 = coop.make_opts()
print("make_opts us", (time.perf_counter() - t) / n * 1e6)
t = time.perf_counter()
for _ in range(n): st, b = coop._stats_struct()
print("stats_struct us", (time.perf_counter() - t) / n * 1e6)
t = time.perf_counter()
for _ in range(n): s = torch.cuda.current_stream().cuda_stream
print("current_stream us", (time.perf_counter() - t) / n * 1e6)
o, k2 = coop.make_opts(); st, b = coop._stats_struct()
t = time.perf_counter()
for _ in range(n): lib.coop_bfs(ctypes.byref(c), 0, out.data_ptr(), ctypes.byref(o), ctypes.byref(st))
print("raw foreign call us", (time.perf_counter() - t) / n * 1e6, "kernel us", st.kernel_ns / 1e3)
t = time.perf_counter()
for _ in range(n): coop._to_runstats(st, b)
print("to_runstats us", (time.perf_counter() - t) / n * 1e6)
