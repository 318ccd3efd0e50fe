"""Build libperiscat_b200.so in-tree with nvcc for sm_100a (no torch dependency).

    python -m paper_1412_7466_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libperiscat_b200.so")
SOURCES = ["m2l.cu", "m2l_mrhs.cu", "m2l_sym.cu", "m2l_symh.cu", "m2l_mma.cu", "coupling.cu", "coupling_dense.cu", "gmres.cu", "field.cu", "empty.cu", "scatmat.cu", "capi.cu", "peak.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]
# The DFMA sweeps of K1s get a post-link SASS scheduling patch
# (sass_reuse_patch.py: operand-reuse flags through the coefficient runs
# instead of ptxas's mid-run yield hints); its device code must therefore sit
# uncompressed in the fatbin.  PS_NO_SASS_PATCH=1 builds the unpatched library.
# Measured per kernel family (tools/probe_patch_gain.py, cfg3): K1s fed by the
# symbol store 1918 -> 1853 us, K1s generating its symbols 2117 -> 2117 us,
# but the tiled K1 2375 -> 2558 us -- its producer warps need the issue slots
# the yields gave them -- so only K1s is patched.
PATCHED_SOURCES = {"m2l_sym.cu"}
PATCHED_KERNELS = r"m2l_sym_(stage_)?kernel"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "periscat_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    if not force and out == LIB and not _stale():
        return LIB
    objs = []
    t0 = time.time()
    procs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", f".{os.getpid()}.o"))
        extra = ["--no-compress"] if src in PATCHED_SOURCES else []
        cmd = [NVCC, *FLAGS, *extra, *[f"-D{d}" for d in defines], "-c",
               os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                            text=True)))
        objs.append(obj)
    log = []
    for src, p in procs:
        txt, _ = p.communicate()
        log.append(f"== {src}\n{txt}")
        if p.returncode != 0:
            sys.stderr.write(txt)
            raise RuntimeError(f"nvcc failed on {src}")
    with open(os.path.join(CSRC, "ptxas.log"), "w") as fh:
        fh.write("\n".join(log))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs,
           "-L/usr/local/cuda/lib64", "-lcusolver", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    try:
        subprocess.run(cmd, check=True)
    finally:                       # no stale objects left behind on a failed link
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    if os.environ.get("PS_NO_SASS_PATCH") != "1":
        stats = sass_patch(out)
        if verbose:
            print(f"SASS reuse patch: {sum(c for _, _, c in stats.values())} DFMAs re-flagged in "
                  f"{len(stats)} kernels")
    if verbose:
        print(f"built {out} in {time.time() - t0:.1f}s")
    return out


def sass_patch(path: str = LIB, dry: bool = False) -> dict:
    """Apply sass_reuse_patch.py to the DFMA kernels of the library;
    returns {kernel: (dfma, already_flagged, patched)}."""
    from . import sass_reuse_patch
    buf = bytearray(open(path, "rb").read())
    stats = sass_reuse_patch.patch(buf, PATCHED_KERNELS)
    if not stats:
        raise RuntimeError("SASS patch: no DFMA kernel found in the fatbin (compressed?)")
    if not dry:
        with open(path, "wb") as fh:
            fh.write(buf)
    return stats


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    build(force="--force" in sys.argv or bool(defs), verbose=True,
          out=outs[0] if outs else LIB, defines=defs)
