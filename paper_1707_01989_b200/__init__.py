"""B200-native cooperative kernels (arXiv 1707.01989): cooperative BFS / SSSP
over CSR in one persistent sm_100a kernel with a resizing global barrier,
offer_kill / request_fork and an in-kernel scheduler.  See DESIGN.md.

The compute path is libcoop.so (include/coop.h); :mod:`.coop` is its thin
ctypes binding and :mod:`.partitioned` the 1-D partitioned multi-GPU driver.
"""
from . import coop  # noqa: F401
from .coop import (CoopError, bfs, sssp, bfs_host, sssp_host, barrier_bench, l2_atomic_rtt,  # noqa: F401
                   device_query, Handle)
