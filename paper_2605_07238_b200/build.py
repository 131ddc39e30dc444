"""Build the sm_100a scorer library in-tree (``paper_2605_07238_b200/libfate.so``).

``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false``.
``--fmad=false`` is part of the exactness contract: it forbids contracting
``a*b+c`` into ``fma.rn.f64``, which would change Psi bits relative to
CPython.  After building, the PTX is scanned and the build fails if any
``fma.rn.f64`` survived outside the walk's tagged exact 0/1-factor blocks.
"""

from __future__ import annotations

import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libfate.so")
SOURCES = [os.path.join(CSRC, "fate_kernels.cu"), os.path.join(CSRC, "fate_host.cpp"),
           os.path.join(CSRC, "fate_synth.cpp"), os.path.join(CSRC, "fate_pipeline.cpp"),
           os.path.join(CSRC, "fate_solver.cpp"), os.path.join(CSRC, "fate_mirror.cu")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-ffp-contract=off", "-I", INCLUDE]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = SOURCES + [os.path.join(INCLUDE, "fate.h"), __file__] + [
        os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return any(os.path.getmtime(p) > t for p in deps)


def check_ptx(verbose: bool = False) -> str:
    """Compile the kernels to PTX and assert no fused multiply-add survived."""
    ptx = os.path.join(HERE, "fate_kernels.ptx")
    cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, "-ptx", SOURCES[0], "-o", ptx]
    subprocess.run(cmd, check=True, capture_output=not verbose)
    if not ptx_contraction_free(open(ptx).read()):
        raise RuntimeError("fma.rn.f64 found in PTX: exactness contract broken")
    return ptx


def ptx_contraction_free(text: str) -> bool:
    """True iff every ``fma.rn.f64`` in the PTX is one of the walk's exact
    0/1-factor FMAs, emitted from inline asm blocks tagged ``fate-fma01``
    (fma(v, 1, a) == v + a and fma(v, 0, a) == a bit for bit); any other is
    a contracted a*b+c."""
    blocks = re.split(r"(// begin inline asm.*?// end inline asm)", text, flags=re.S)
    rest = "".join(b for b in blocks
                   if not (b.startswith("// begin inline asm") and "fate-fma01" in b))
    return re.search(r"\bfma\.rn\.f64\b", rest) is None


def ab_build() -> bool:
    """FATE_BUILD_AB=1: experiment build with the previous kernel generation
    and the environment A/B knobs compiled in (-DFATE_AB).  Production builds
    run exactly one kernel generation with the measured launch shape."""
    return os.environ.get("FATE_BUILD_AB", "") not in ("", "0")


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    tmp = LIB + ".tmp"
    extra = ["-DFATE_AB"] if ab_build() else []
    # experiment-only preprocessor defines (A/B of kernel variants), e.g.
    # FATE_BUILD_DEFS="FATE_V6_NOPF"
    extra += ["-D" + d for d in os.environ.get("FATE_BUILD_DEFS", "").split()]
    extra += os.environ.get("FATE_BUILD_NVCC", "").split()  # experiment-only nvcc flags
    cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, *extra, "-shared", "-Xptxas", "-v", *SOURCES, "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libfate.so")
    if verbose:
        sys.stderr.write(res.stderr)
    with open(os.path.join(HERE, "libfate.ptxas.txt"), "w") as fh:
        fh.write(res.stderr)
    os.replace(tmp, LIB)
    check_ptx()
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
