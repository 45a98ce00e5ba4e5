"""Build an A/B variant of libparadyse.so with extra nvcc defines for ONE source file
(e.g. the attention kernels), linked with the regular objects of the others:

  python tools/build_variant.py attn_tc.cu --define PDS_EMU_MASK=0x00 --out build/variants/emu00.so
  PDS_LIB=build/variants/emu00.so python bench.py ...
"""
import argparse
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_13198_b200 import build as Bd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("source")
    ap.add_argument("--define", action="append", default=[])
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    Bd.build()
    nd = Bd.nccl_dir()
    src = [s for s in Bd.sources() if s.endswith(a.source)][0]
    os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
    obj = a.out + ".o"
    subprocess.run([Bd.nvcc(), *Bd.ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3",
                    "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"), *["-D" + d for d in a.define],
                    "-c", src, "-o", obj], check=True)
    rel = os.path.relpath(src, Bd.CSRC).replace(os.sep, "_") + ".o"
    objs = [o for o in glob.glob(os.path.join(Bd.BUILD, "*.o")) if os.path.basename(o) != rel] + [obj]
    lib = os.path.join(nd, "lib")
    subprocess.run([Bd.nvcc(), *Bd.ARCH, "-shared", "-o", a.out, *objs, "-L", lib, "-l:libnccl.so.2",
                    "-Xlinker", f"-rpath,{lib}", "-lcudart_static", "-lpthread", "-ldl", "-lrt"], check=True)
    print(a.out)


if __name__ == "__main__":
    main()
