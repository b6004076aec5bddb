"""CPU checks of the boundary: libcoop.so builds for sm_100a, loads, and
exports every function include/coop.h declares (no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "coop.h")


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(coop_[a-z_0-9]+)\s*\(", text, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1707_01989_b200 import build
    return build.build()


def test_header_declares_the_north_star_entry_points():
    names = _declared_functions()
    for n in ["coop_bfs", "coop_sssp", "coop_launch", "coop_submit_task", "coop_demand", "coop_grant",
              "coop_query", "coop_wait", "coop_barrier_bench", "coop_bfs_host", "coop_sssp_host"]:
        assert n in names
    for n in ["coop_dev_create", "coop_dev_arm", "coop_dev_demand", "coop_dev_grant", "coop_dev_collect",
              "coop_dev_destroy", "coop_fig4_bfs", "coop_work_steal"]:
        assert n in names
    for n in ["coop_bfs_part", "coop_bfs_part_nccl", "coop_nccl_get_unique_id", "coop_nccl_comm_init",
              "coop_nccl_comm_destroy"]:
        assert n in names
    assert "coop_bfs_loop" in names
    assert len(names) == 50


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    missing = [n for n in _declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    for n in _declared_functions():
        assert re.search(rf"\bT {n}\b", out), n


def test_binding_covers_header(lib_path):
    from paper_1707_01989_b200 import coop
    assert sorted(coop.SIGNATURES) == _declared_functions()
    lib = coop.load(lib_path)
    assert lib.coop_abi_version() == 1
    assert lib.coop_status_string(6) == b"COOP_ERR_TIMEOUT"
    assert lib.coop_status_string(0) == b"COOP_OK"


def test_struct_layouts_match_header(lib_path):
    """ctypes mirrors of the C structs: sizes computed by the C compiler."""
    from paper_1707_01989_b200 import coop
    src = """
#include <stdio.h>
#include <stddef.h>
#include "coop.h"
int main(void){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(coop_csr), sizeof(coop_opts),
 sizeof(coop_stats), sizeof(coop_task_event), sizeof(coop_device_info), sizeof(coop_barrier_stats),
 sizeof(coop_part), sizeof(coop_dev_opts), sizeof(coop_dev_stats), sizeof(coop_ws_tree), sizeof(coop_ws_result));
 return 0;}
"""
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "s.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "s")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, c])
        sizes = [int(x) for x in subprocess.check_output([exe]).split()]
    assert sizes == [ctypes.sizeof(t) for t in (coop.CooperativeCSR, coop.Opts, coop.Stats, coop.TaskEvent,
                                                coop.DeviceInfo, coop.BarrierStats, coop.CoopPart,
                                                coop.DevOpts, coop.DevStats, coop.WsTree, coop.WsResult)]


def test_sass_targets_sm100a(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_invalid_args_fail_cleanly_without_gpu(lib_path):
    """Argument validation happens before any device work: NULL graph -> INVALID_ARG."""
    from paper_1707_01989_b200 import coop
    lib = coop.load(lib_path)
    rc = lib.coop_bfs(None, 0, None, None, None)
    assert rc in (1, 2)          # INVALID_ARG, or CUDA if no driver is present at all
    assert lib.coop_last_error()


def test_device_api_header_compiles_in_a_user_kernel(tmp_path):
    """include/coop_device.cuh is self-contained: a user kernel using every
    device entry point (offer_kill, request_fork, global_barrier,
    resizing_global_barrier, group id / count, query, transmit) and the host
    launch helper compiles for sm_100a."""
    src = tmp_path / "user.cu"
    src.write_text(r"""
#include "coop_device.cuh"
struct T { unsigned level; };
__global__ void user_kernel(coop_dev *d, int *out) {
    coop_run(d, [&](coop_ctx *c) {
        T t = {0};
        if (coop_entry(c)) coop_get_transmit(c, &t, sizeof t);
        for (;;) {
            if (coop_offer_kill(c)) return;
            coop_request_fork(c, &t, sizeof t, 1);
            if (threadIdx.x == 0) atomicAdd(out + coop_group_id(c) % 4, (int)coop_num_groups(c) + (int)coop_query_dev(c));
            if (!coop_global_barrier(c)) return;
            t.level++;
            if (!coop_resizing_global_barrier(c, &t, sizeof t, 1)) return;
            if (t.level > 3) return;
        }
    });
}
int launch(coop_dev *d, int *out) {
    unsigned n = 0;
    coop_dev_max_wgs(user_kernel, 128, 0, &n);
    return (int)coop_dev_launch(user_kernel, n, 128, 0, (cudaStream_t)0, d, out);
}
""")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17",
                           "-I", os.path.join(ROOT, "include"), "-c", "-o", str(tmp_path / "user.o"), str(src)])
