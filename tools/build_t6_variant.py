"""A/B helper: relink libsfseg.so with only spass_tc6.cu recompiled under extra defines.

    python tools/build_t6_variant.py OUT.so -DT6_LDALL=0 -DT6_L2PF=0

Needs the objects of a product build in build/ (run __graft_entry__.build() first).  The
variant library is written to OUT.so; copy it over paper_2212_08058_b200/libsfseg.so to use it.
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2212_08058_b200 import build as B  # noqa: E402


def main():
    out, defs = sys.argv[1], sys.argv[2:]
    nvcc = B._nvcc()
    obj = os.path.join(B.BUILD, "spass_tc6_variant.o")
    r = subprocess.run([nvcc, *B.ARCH, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, "spass_tc6.cu"), "-o", obj],
                       capture_output=True, text=True)
    if r.returncode != 0:
        sys.exit(r.stderr)
    objs = [os.path.join(B.BUILD, s.replace(".cu", ".o")) for s in B.SOURCES if s != "spass_tc6.cu"] + [obj]
    r = subprocess.run([nvcc, *B.ARCH, "-shared", "-o", out, *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        sys.exit(r.stderr)
    print(out)


if __name__ == "__main__":
    main()
