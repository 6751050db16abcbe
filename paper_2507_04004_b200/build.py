"""Build the sm_100a extension in-tree: paper_2507_04004_b200/lib/libgslic.so.

    python -m paper_2507_04004_b200.build [--force]

nvcc compiles every csrc/*.cu for `-gencode arch=compute_100a,code=sm_100a` with -lineinfo
(so ncu source pages map to the code) and links one shared library exposing the C ABI of
include/gslic.h.  No torch headers are involved: the ABI is plain pointers and sizes.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libgslic.so")
SOURCES = ["api.cu", "preprocess.cu", "binning.cu", "render.cu", "loss.cu", "adam.cu", "keyframe.cu", "track.cu",
           "p2p.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in os.listdir(CSRC)
                                                      if h.endswith(".cuh")] + [os.path.join(ROOT, "include", "gslic.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile and link libgslic.so (or, with `defines` / `out`, an experiment variant elsewhere)."""
    if not force and not defines and out is None and not _stale():
        return LIB
    lib_out = out or LIB
    objdir = os.path.join(LIBDIR, "obj") if out is None else os.path.join(os.path.dirname(out), "obj_" + os.path.basename(out))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    logs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        objs.append(obj)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib_out, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    if out is None:
        with open(os.path.join(LIBDIR, "ptxas.log"), "w") as fh:
            fh.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return lib_out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, out=outs[0] if outs else None))
