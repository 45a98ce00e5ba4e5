"""Build libparadyse.so (sm_100a) in-tree with nvcc.

All CUDA kernels and the C++ host library compile into one shared object
`paper_2511_13198_b200/libparadyse.so` exporting the C ABI of include/paradyse.h.
NCCL is the torch wheel's 2.28.x (header + libnccl.so.2) so one process never
loads two NCCLs.  Objects are cached under build/ keyed by source mtime.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import site
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libparadyse.so")
BUILD = os.path.join(ROOT, "build", "obj")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir():
    for sp in site.getsitepackages() + [site.getusersitepackages()]:
        d = os.path.join(sp, "nvidia", "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("torch's NCCL wheel (nvidia/nccl) not found")


def nvcc():
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cpp")) + glob.glob(os.path.join(CSRC, "kernels", "*.cu")))


def headers_mtime():
    hs = glob.glob(os.path.join(CSRC, "**", "*.h*"), recursive=True) + \
        glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True) + \
        [os.path.join(ROOT, "include", "paradyse.h")]
    return max(os.path.getmtime(h) for h in hs)


def compile_one(src, nd, verbose=False):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    obj = os.path.join(BUILD, rel + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), headers_mtime()):
        return obj
    cmd = [nvcc(), *ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"),
           "-c", src, "-o", obj]
    if src.endswith(".cu"):
        cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
    else:
        cmd += ["-x", "cu"] if False else []
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose=False, force=False):
    os.makedirs(BUILD, exist_ok=True)
    nd = nccl_dir()
    srcs = sources()
    if force:
        for f in glob.glob(os.path.join(BUILD, "*.o")):
            os.remove(f)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: compile_one(s, nd, verbose), srcs))
    newest = max(os.path.getmtime(o) for o in objs)
    if os.path.exists(OUT) and os.path.getmtime(OUT) >= newest and not force:
        return OUT
    lib = os.path.join(nd, "lib")
    cmd = [nvcc(), *ARCH, "-shared", "-o", OUT, *objs, "-L", lib, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath,{lib}", "-lcudart_static", "-lpthread", "-ldl", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
