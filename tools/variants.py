"""Builds experiment variants of the product library: one source file
recompiled with extra -D flags, linked with the other objects of the normal
build, into paper_2203_09087_b200/lib/variants/<name>.so.  Select one at run
time with ECC_B200_LIB=<path>.  Tooling for kernel experiments only.

  python tools/variants.py k_u8_3d.cu base= pred=-DECC_U83D_PRED_ATOMS=1
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2203_09087_b200 import build as B  # noqa: E402


def main():
    src = sys.argv[1]
    B.build()
    objdir = os.path.join(B.LIBDIR, "obj")
    vdir = os.path.join(B.LIBDIR, "variants")
    os.makedirs(vdir, exist_ok=True)
    others = [os.path.join(objdir, os.path.basename(s) + ".o") for s in B.sources()
              if os.path.basename(s) != src]
    procs = []
    for spec in sys.argv[2:]:
        name, _, flags = spec.partition("=")
        obj = os.path.join(vdir, f"{name}.o")
        cmd = [B.NVCC, *B.ARCH, *B.FLAGS, *flags.split(), "-c", os.path.join(B.CSRC, src), "-o", obj]
        procs.append((name, obj, subprocess.Popen(cmd)))
    for name, obj, p in procs:
        if p.wait() != 0:
            sys.exit(f"variant {name} failed to compile")
        so = os.path.join(vdir, f"{name}.so")
        subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", so, obj, *others, "-Xcompiler", "-fPIC"],
                       check=True)
        print(so)


if __name__ == "__main__":
    main()
