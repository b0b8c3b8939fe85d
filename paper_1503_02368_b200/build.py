"""Build libeh.so (CUDA, sm_100a) in-tree with nvcc.

``python -m paper_1503_02368_b200.build`` or ``__graft_entry__.build()``.
The .so lands in paper_1503_02368_b200/lib/ so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import glob
import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIBDIR = os.path.join(PKG, "lib")
SO = os.path.join(LIBDIR, "libeh.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
              "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _digest() -> str:
    h = hashlib.sha256()
    for f in sorted(_sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "eh.h"),
                                                                            os.path.abspath(__file__)]):
        h.update(f.encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


SO_CHECKED = os.path.join(LIBDIR, "libeh_checked.so")


def build(force: bool = False, verbose: bool = False, jobs: int | None = None, checked: bool = False) -> str:
    """Compile every csrc/*.cu to an object (in parallel) and link libeh.so.

    checked=True builds lib/libeh_checked.so instead: the same sources with
    -DEH_CHECKED, i.e. the device-side bounds assertions of csrc/check.cuh live
    (the test suite's substitute for compute-sanitizer, closed on this pool)."""
    os.makedirs(LIBDIR, exist_ok=True)
    so = SO_CHECKED if checked else SO
    stamp = os.path.join(LIBDIR, "libeh_checked.sha256" if checked else "libeh.sha256")
    dig = _digest()
    if not force and os.path.exists(so) and os.path.exists(stamp) and open(stamp).read().strip() == dig:
        return so
    objdir = os.path.join(LIBDIR, "obj_checked" if checked else "obj")
    os.makedirs(objdir, exist_ok=True)
    cc = nvcc()
    procs = []
    objs = []
    for src in _sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        cmd = [cc, *ARCH, *NVCC_FLAGS, *(["-DEH_CHECKED"] if checked else []), "-I", INCLUDE, "-I", CSRC,
               "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        txt = out.decode(errors="replace")
        if p.returncode != 0:
            failed.append((src, txt))
        elif verbose and txt.strip():
            print(txt)
    if failed:
        msg = "\n".join(f"--- {s}\n{t}" for s, t in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    tmp = so + f".tmp{os.getpid()}"
    subprocess.check_call([cc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"])
    os.replace(tmp, so)
    with open(stamp, "w") as f:
        f.write(dig)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
