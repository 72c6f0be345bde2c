"""Build libpfc.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, os.environ.get("PFC_LIB_NAME", "libpfc.so"))
SOURCES = ["pfc.cu", "stencil2d.cu", "stencil3d.cu", "krylov.cu", "energy.cu", "ras2d.cu",
           "ras3d.cu", "ras3d_col.cu", "ras3d_cl2.cu", "ras_extend.cu", "mobility.cu",
           "ilu.cu", "tail2d.cu", "newton_graph.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]
FLAGS += os.environ.get("PFC_EXTRA_NVCC_FLAGS", "").split()   # diagnostic builds only


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "pfc.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "..", "build", "obj" + os.environ.get("PFC_LIB_NAME", ""))
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)

    # diagnostic variants (PFC_LIB_NAME + PFC_EXTRA_NVCC_FLAGS) may recompile only the sources
    # listed in PFC_VARIANT_SOURCES and reuse the default build's objects for the rest
    only = [f for f in os.environ.get("PFC_VARIANT_SOURCES", "").split(",") if f]
    basedir = os.path.join(HERE, "..", "build", "obj")

    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if not f.endswith(".cu")]
    headers.append(os.path.join(HERE, "..", "include", "pfc.h"))
    hdr_t = max(os.path.getmtime(h) for h in headers)

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        if only and src not in only:
            base = os.path.join(basedir, src.replace(".cu", ".o"))
            if os.path.exists(base):
                return base, ""
        # incremental: an object newer than its source and every header is reused
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(
                os.path.getmtime(os.path.join(CSRC, src)), hdr_t):
            return obj, ""
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log = "\n".join(r[1] for r in results)
    with open(os.path.join(objdir, "ptxas.log"), "w") as f:
        f.write(log)
    if verbose:
        print(log)
    objs = [r[0] for r in results]
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           "-o", LIB, *objs]
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
