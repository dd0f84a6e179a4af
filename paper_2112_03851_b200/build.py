"""Builds libosm.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo snapshot).

    python paper_2112_03851_b200/build.py [--verbose-ptxas] [--force]   (or __graft_entry__.build())
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libosm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import nvidia.nccl  # torch's bundled NCCL (2.28): headers + libnccl.so.2

    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("command failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def gen_kuhn_slots(force: bool = False) -> str:
    """Generated header kuhn_slots.h: the P2 Kuhn stencil slots per parity class, computed by the
    library's own host geometry (csrc/gen_kuhn_slots.cpp + lattice.cpp) for the brick SpMV."""
    out = os.path.join(OBJ, "kuhn_slots.h")
    deps = [os.path.join(CSRC, f) for f in ("gen_kuhn_slots.cpp", "lattice.cpp", "lattice.h")]
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps):
        return out
    exe = os.path.join(OBJ, "gen_kuhn_slots")
    _run([os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-I", CSRC, "-I", INCLUDE, "-I", "/usr/local/cuda/include",
          deps[0], deps[1], "-o", exe])
    r = subprocess.run([exe], capture_output=True, text=True, check=True)
    with open(out + ".tmp", "w") as f:
        f.write(r.stdout)
    os.replace(out + ".tmp", out)
    return out


def build(verbose_ptxas: bool = False, force: bool = False) -> str:
    inc, lib = nccl_dirs()
    os.makedirs(OBJ, exist_ok=True)
    gen_kuhn_slots(force)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) +
                  [f for f in glob.glob(os.path.join(CSRC, "*.cpp")) if not os.path.basename(f).startswith("gen_")])
    headers = glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(INCLUDE, "osm.h"), os.path.join(OBJ, "kuhn_slots.h")]
    newest_header = max(os.path.getmtime(h) for h in headers)
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC, "-I", OBJ, "-I", inc,
             "--expt-relaxed-constexpr"] + ARCH
    if verbose_ptxas:
        flags += ["-Xptxas", "-v"]
    jobs = []
    objs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s) + ".o")
        objs.append(o)
        if force or verbose_ptxas or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), newest_header):
            jobs.append([NVCC, "-c", s, "-o", o] + flags)
    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for out in ex.map(_run, jobs):
            logs.append(out)
    if jobs or not os.path.exists(LIB):
        _run([NVCC, "-shared", "-o", LIB] + objs + ARCH +
             ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib])
    return "\n".join(logs)


if __name__ == "__main__":
    out = build(verbose_ptxas="--verbose-ptxas" in sys.argv, force="--force" in sys.argv)
    if out.strip():
        print(out)
    print("built", LIB)
