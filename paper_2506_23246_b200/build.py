"""Build the in-tree CUDA library ``libqpinn_b200.so`` for sm_100a.

nvcc cross-compiles without a GPU, so this runs in the CPU build container
(``__graft_entry__.build()``) and the resulting .so travels to the GPU box
with the repository snapshot.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libqpinn_b200.so")
SOURCES = (["circuit.cu", "pqc.cu", "pqc_layer.cu", "pqc_layer_f64.cu", "pqc_big_dispatch.cu", "trunk.cu", "loss.cu",
            "adam.cu", "tc_gemm.cu", "fdtd.cu", "probes.cu", "pqc_global.cu", "pqc_transfer.cu"] + [f"pqc_big_n{n}.cu" for n in range(9, 17)])
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def _stamp():
    h = hashlib.sha256()
    for f in sorted(os.listdir(CSRC)) + ["../../include/qpinn_b200.h"]:
        path = os.path.normpath(os.path.join(CSRC, f))
        if os.path.isfile(path) and f.endswith((".cu", ".cuh", ".h")):
            h.update(f.encode())
            with open(path, "rb") as fh:
                h.update(fh.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    stamp_file = LIB + ".stamp"
    stamp = _stamp()
    if not force and os.path.exists(LIB) and os.path.exists(stamp_file):
        with open(stamp_file) as f:
            if f.read().strip() == stamp:
                return LIB
    nvcc = _nvcc()
    objs = []
    logs = []
    procs = []
    # per-source object cache: a source is recompiled only when it, a header or the flags change
    odir = os.path.join(CSRC, ".obj")
    os.makedirs(odir, exist_ok=True)
    hdr = hashlib.sha256()
    for f in sorted(os.listdir(CSRC)) + ["../../include/qpinn_b200.h"]:
        if f.endswith((".h", ".cuh")):
            with open(os.path.normpath(os.path.join(CSRC, f)), "rb") as fh:
                hdr.update(f.encode() + fh.read())
    hdr.update(" ".join(ARCH + FLAGS).encode())
    for src in SOURCES:
        with open(os.path.join(CSRC, src), "rb") as fh:
            key = hashlib.sha256(hdr.digest() + fh.read()).hexdigest()[:16]
        obj = os.path.join(odir, src.replace(".cu", f".{key}.o"))
        if os.path.exists(obj):
            objs.append(obj)
            continue
        cmd = [nvcc, *ARCH, *FLAGS, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
               "-c", os.path.join(CSRC, src), "-o", obj + ".tmp"]
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                 stderr=subprocess.PIPE, text=True)))
    for src, obj, pr in procs:
        out, err = pr.communicate()
        logs.append(err)
        if pr.returncode != 0:
            sys.stderr.write(out + err)
            raise RuntimeError(f"nvcc failed on {src}")
        os.replace(obj + ".tmp", obj)
        objs.append(obj)
    keep = set(objs)
    for f in os.listdir(odir):
        if os.path.join(odir, f) not in keep:
            os.remove(os.path.join(odir, f))
    tmp = LIB + ".tmp"
    cmd = [nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-lcublas",
           "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, LIB)
    if logs:
        with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
            f.write("\n".join(logs))
    with open(stamp_file, "w") as f:
        f.write(stamp)
    if verbose:
        print("built", LIB)
    return LIB



TOOLS_LIB = os.path.join(HERE, "libqpinn_tools.so")


def build_tools(verbose: bool = False) -> str:
    """Microbenchmarks used by bench.py (not part of the QPINN ABI)."""
    src = os.path.join(CSRC, "tools", "fp32_peak.cu")
    if os.path.exists(TOOLS_LIB) and os.path.getmtime(TOOLS_LIB) > os.path.getmtime(src):
        return TOOLS_LIB
    cmd = [_nvcc(), *ARCH, "-O3", "-Xcompiler", "-fPIC", "-shared", src, "-o", TOOLS_LIB]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("tools build failed")
    if verbose:
        print("built", TOOLS_LIB)
    return TOOLS_LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    build_tools(verbose=True)
