"""Build libkvshare.so with extra nvcc defines into a given path (experiments).

    python tools/build_variant.py /tmp/libkvs_x.so -DKVS_POLY_EVERY=2 ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_16525_b200 import build as B  # noqa: E402

out, defs = sys.argv[1], sys.argv[2:]
objs = []
for src in B.SOURCES:
    o = f"{out}.{src}.o"
    subprocess.check_call([B.NVCC, *B.ARCH, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", o])
    objs.append(o)
subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", out, *objs, "-lcudart_static"])
print(out)
