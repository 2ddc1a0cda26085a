"""Build libgk.so (the C-ABI product library) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libgk.so")
SOURCES = ["gk_api.cu", "gk_encode.cu", "gk_filter.cu", "gk_filter_ascii.cu", "gk_compact.cu",
           "gk_filter_ascii_p0.cu", "gk_filter_ascii_p1.cu", "gk_filter_ascii_p2.cu",
           "gk_filter_ascii_p3.cu", "gk_filter_bt2.cu", "gk_filter_sp2.cu", "gk_fused.cu", "gk_verify.cu", "gk_index.cu"]
HEADERS = ["gk_common.cuh", "gk_kernels.cuh", "gk_encode_core.cuh", "gk_filter_core.cuh",
           "gk_tma.cuh", "gk_filter_ascii_impl.cuh", "gk_encode3.cuh", "gk_bt2.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _inputs():
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "gatekeeper.h"))
    files.append(os.path.abspath(__file__))
    return files


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in _inputs())


def build(verbose: bool = False, force: bool = False, jobs: int | None = None,
          defines=(), out: str | None = None) -> str:
    """Build libgk.so (or, with `defines` such as ["GK_BT2_B=16"], an A/B variant at `out`)."""
    so = out or SO
    if not force and not defines and not stale():
        return SO
    if defines and os.path.exists(so) and not force:
        t = os.path.getmtime(so)
        if all(os.path.getmtime(f) <= t for f in _inputs()):
            return so
    objdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(
        d.replace("=", "") for d in defines))
    os.makedirs(objdir, exist_ok=True)
    common = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
    common += [f"-D{d}" for d in defines]
    if verbose:
        common += ["-Xptxas", "-v"]
    procs, objs = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = common + ["-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                            stderr=subprocess.STDOUT, text=True)))
    failed = False
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"[gk build] FAILED: {' '.join(cmd)}\n{out}\n")
        elif verbose and out:
            sys.stderr.write(out)
    if failed:
        raise RuntimeError("libgk.so build failed")
    link = ["nvcc", *ARCH, "-shared", "-cudart", "shared", "-Xlinker",
            "-rpath,/usr/local/cuda/lib64", "-o", so, *objs]
    subprocess.check_call(link)
    return so


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(SO)
