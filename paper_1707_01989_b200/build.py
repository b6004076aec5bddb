"""Build libcoop.so in-tree with nvcc for sm_100a (no GPU needed to build).

    python -m paper_1707_01989_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcoop.so")
SOURCES = [os.path.join(CSRC, f) for f in ("coop_api.cu", "coop_dev_api.cu", "coop_layout.cu")]
DEPS = SOURCES + sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))) + \
    [os.path.join(ROOT, "include", f) for f in ("coop.h", "coop_device.cuh", "coop_protocol.cuh")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-shared",
]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    if not force and out == LIB and not needs_build():
        return LIB
    # one nvcc per translation unit, in parallel (separate TUs either way: no -rdc), then link
    common = [NVCC, *FLAGS[:-1], *(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines]]
    objs = [f"{out}.{os.path.basename(s)}.o" for s in SOURCES]

    def compile_one(i):
        return subprocess.run([*common, "-c", "-o", objs[i], SOURCES[i]], capture_output=True, text=True)

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(compile_one, range(len(SOURCES))))
    results.append(subprocess.run([NVCC, *FLAGS, "-o", out + ".tmp", *objs], capture_output=True, text=True)
                   if all(r.returncode == 0 for r in results) else results[0])
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    for res in results:
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
        if verbose:
            sys.stderr.write(res.stderr)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv or bool(defs), verbose="--verbose" in sys.argv,
                out=outs[0] if outs else LIB, defines=defs))
