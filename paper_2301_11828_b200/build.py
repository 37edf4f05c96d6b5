"""Build libpdgpu.so (the CUDA engine + C ABI) in-tree for sm_100a.

    python -m paper_2301_11828_b200.build        # or build() from __graft_entry__

Explicit nvcc invocation; no torch extension machinery.  The library is a
plain C-ABI shared object loaded with ctypes (paper_2301_11828_b200/_lib.py).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpdgpu.so")
# spectral.cu is compiled once per part (-DPDGPU_PART=k): each object
# instantiates only its own kernel templates, and the parts build in parallel
SPECTRAL_PARTS = 5
SOURCES = ["spectral.cu", "corrections.cu", "direct.cu", "solvers.cu", "abi.cu", "transpose.cu", "assembly.cpp",
           "snapshot.cpp", "comm.cpp"]
HEADERS = ["engine.h", "fft.cuh", "assembly.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off", "--expt-relaxed-constexpr"]


def _inputs():
    files = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    files.append(os.path.join(HERE, "..", "include", "pdgpu.h"))
    files.append(os.path.abspath(__file__))
    return files


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _inputs() if os.path.exists(f))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    units = []
    for s in SOURCES:
        if s == "spectral.cu":
            units += [(s, f"{s}.part{k}.o", [f"-DPDGPU_PART={k}"]) for k in range(SPECTRAL_PARTS)]
        elif s == "corrections.cu":
            units.append((s, s + ".o", ["--fmad=false"]))  # bond stretch must round like the reference
        else:
            units.append((s, s + ".o", []))
    for s, oname, extra in units:
        src = os.path.join(CSRC, s)
        obj = os.path.join(objdir, oname)
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd) + "\n" + out.decode())
        if verbose:
            sys.stdout.write(out.decode())
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed: " + r.stdout + r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
