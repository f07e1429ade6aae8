"""Build the native libraries in-tree (``python -m paper_2512_04389_b200.build``).

* liblbk_host.so — g++ -O3, structure path (csrc/lbk_host.cpp)
* liblbk.so      — nvcc for sm_100a (-gencode arch=compute_100a,code=sm_100a),
                   device engine (csrc/lbk_device.cu), links cudart statically
                   so the .so only needs the driver on the GPU box.

Outputs land in paper_2512_04389_b200/_lib (git-ignored, travels with gpurun).

Checker only (never imported by the package): where /root/reference exists,
the unmodified reference is pip-installed into baseline/_ref (git-ignored,
travels with gpurun) for the CPU-reference timing (oracle/ref_timing.py) and
the golden fixtures.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_lib")
INC = os.path.join(os.path.dirname(PKG), "include")

NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


REF_SRC = "/root/reference/pkg"
REF_DST = os.path.join(os.path.dirname(PKG), "baseline", "_ref")


def install_reference(verbose: bool = False) -> None:
    """pip install --no-index --target baseline/_ref of the read-only reference (built from a /tmp copy)."""
    if not os.path.isdir(REF_SRC) or os.path.isdir(os.path.join(REF_DST, "lublock")):
        return
    import tempfile

    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_SRC, src)
        _run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
              "--find-links", "/opt/wheelhouse", "--target", REF_DST, "-q", src], verbose)


def build(verbose: bool = False, force: bool = False) -> None:
    install_reference(verbose)
    os.makedirs(OUT, exist_ok=True)
    hdr = os.path.join(INC, "lbk.h")
    host_src = os.path.join(SRC, "lbk_host.cpp")
    host_out = os.path.join(OUT, "liblbk_host.so")
    if force or _stale(host_out, [host_src, hdr]):
        _run(["g++", "-O3", "-std=c++17", "-fPIC", "-shared", "-Wall", "-I", INC,
              "-o", host_out, host_src], verbose)
    dev_srcs = [os.path.join(SRC, f) for f in sorted(os.listdir(SRC)) if f.endswith(".cu")]
    dev_out = os.path.join(OUT, "liblbk.so")
    deps = dev_srcs + [hdr] + [os.path.join(SRC, f) for f in os.listdir(SRC) if f.endswith(".cuh")]
    if force or _stale(dev_out, deps):
        _run([_nvcc(), *NVCC_ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-shared", "-cudart", "static", "-Xptxas", "-v" if verbose else "-O3", "-I", INC,
              "-o", dev_out, *dev_srcs], verbose)


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
