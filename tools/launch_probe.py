"""Launch + teardown cost of the persistent cooperative kernel: barrier benchmark with 1 barrier
(event time around the kernel vs the kernel's own %globaltimer window)."""
from paper_1707_01989_b200 import coop
for n in (148, 296, 592, 1184):
    for thr in (128, 512):
        if (thr == 512 and n > 296) or n * thr > 148 * 2048:
            continue
        rs = [coop.barrier_bench(n, 1, threads=thr, plain=True) for _ in range(5)]
        print(n, thr, "event_ns", [round(r["ns_per_barrier"]) for r in rs[1:]], "kernel_ns", [r["kernel_ns"] for r in rs[1:]])
