"""Dev tool: build libqpinn_b200 variants with extra nvcc -D flags for one
translation unit (kernel tuning experiments).  Output: exp/<tag>.so, loaded
by setting QPINN_LIB_OVERRIDE.  Usage: build_variant.py <tag> <src.cu> -DNAME=V ..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_23246_b200 import build as B  # noqa: E402

tag, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
odir = os.path.join(B.CSRC, ".obj")
objs = [os.path.join(odir, f) for f in os.listdir(odir)
        if f.endswith(".o") and not f.startswith(src.replace(".cu", "."))]
os.makedirs(os.path.join(B.ROOT, "exp"), exist_ok=True)
obj = os.path.join(B.ROOT, "exp", f"{tag}.o")
subprocess.run([B._nvcc(), *B.ARCH, *B.FLAGS, *defs, "-I", os.path.join(B.ROOT, "include"),
                "-I", B.CSRC, "-c", os.path.join(B.CSRC, src), "-o", obj], check=True,
               capture_output=True)
subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", os.path.join(B.ROOT, "exp", f"{tag}.so"),
                *objs, obj, "-lcudart", "-lcublas", "-Xlinker", "-rpath,/usr/local/cuda/lib64"],
               check=True)
os.remove(obj)
print("built", tag)
