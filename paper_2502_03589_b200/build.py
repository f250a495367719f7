"""Build libhack.so in-tree with nvcc for sm_100a (B200).

    python paper_2502_03589_b200/build.py          # incremental
    python paper_2502_03589_b200/build.py --force  # rebuild everything
(run by path: importing the package needs the library it builds)

Objects go to paper_2502_03589_b200/build/, the library to
paper_2502_03589_b200/libhack.so (git-ignored, travels with gpurun snapshots).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libhack.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          "--expt-relaxed-constexpr", "-Xptxas", "-v,-warn-spills"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec else []
    for r in roots:
        inc, lib = os.path.join(r, "nccl", "include"), os.path.join(r, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("NCCL headers not found (expected site-packages/nvidia/nccl)")


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    inc, libdir = nccl_dirs()
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "hack.h")]
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = []
    objs = []
    extra = os.environ.get("HACK_EXTRA_NVCC_FLAGS", "").split()  # experiments only
    for s in sources:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        cmd = [NVCC, *ARCH, *CFLAGS, *extra, "-I", inc, "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o]
        # the object's compile flags are stamped next to it: a flag change (e.g. an ablation
        # build with HACK_EXTRA_NVCC_FLAGS left behind) forces a rebuild, not just an mtime change
        stamp = o + ".flags"
        old = open(stamp).read() if os.path.exists(stamp) else None
        if force or _newer([s] + headers, o) or old != " ".join(cmd):
            jobs.append((s, cmd))

    def run(job):
        s, cmd = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        return s, r, cmd

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for s, r, cmd in ex.map(run, jobs):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {os.path.basename(s)}")
            if verbose:
                sys.stderr.write(f"== {os.path.basename(s)}\n" + r.stderr)
            with open(os.path.join(BUILD, os.path.basename(s) + ".ptxas.txt"), "w") as f:
                f.write(r.stderr)
            with open(os.path.join(BUILD, os.path.basename(s) + ".o.flags"), "w") as f:
                f.write(" ".join(cmd))
    if force or jobs or _newer(objs, LIB):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-L", libdir, "-l:libnccl.so.2",
               "-Xlinker", f"-rpath={libdir}", "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
