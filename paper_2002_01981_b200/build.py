"""Build libpifcm.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2002_01981_b200.build [--force]

The library statically links the CUDA runtime so it does not depend on the
runtime version torch ships; device pointers and streams from torch are valid
in it (same driver context).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpifcm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-I", os.path.join(ROOT, "include")]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None,
          only=()) -> str:
    """Compile every csrc/*.cu for sm_100a and link libpifcm.so.  `defines` /
    `out` build tuning variants (e.g. PIFCM_RING=6) under another name; with
    `only` (source basenames) just those sources take the defines and the
    other objects come from the default build."""
    lib = out or LIB
    if not force and not defines and out is None and not needs_build():
        return LIB
    objdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(d.replace("=", "") for d in defines))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    # per object: recompile when the object is missing or older than its
    # source, any header or this script (headers are not tracked per source)
    hdr_t = max([os.path.getmtime(f) for f in headers()] + [os.path.getmtime(__file__)])
    for src in sources():
        if only and os.path.basename(src) not in only:
            objs.append(os.path.join(HERE, "build", os.path.basename(src) + ".o"))
            continue
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(os.path.getmtime(src), hdr_t):
            continue
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-Xptxas", "-v" if verbose else "-O3",
               "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{out.decode()}")
        if verbose:
            sys.stdout.write(out.decode())
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lrt", "-ldl", "-lpthread"]
    out = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if out.returncode != 0:
        raise RuntimeError(f"link failed:\n{out.stdout.decode()}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    only = [s for a in sys.argv[1:] if a.startswith("--only=") for s in a[7:].split(",")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                out=outs[0] if outs else None, only=only))
