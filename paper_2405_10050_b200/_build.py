"""In-tree nvcc build of the C-ABI shared library (sm_100a only).

The library is a plain ``extern "C"`` shared object (``include/voronray_b200.h``)
compiled with nvcc for ``-gencode arch=compute_100a,code=sm_100a`` and the
CUDA runtime linked statically, so it does not depend on torch's bundled
runtime.  It is loaded with ctypes by :mod:`paper_2405_10050_b200._lib`.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_NAME = "_voronray_b200.so"
LIB_PATH = os.path.join(PKG_DIR, LIB_NAME)

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--cudart", "static",
]


def _nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the B200 library cannot be built")


def _npyrandom():
    """NumPy's static distribution library (random_standard_normal): the
    host descent streams (csrc/host_rng.cu) draw with NumPy's own ziggurat so
    that they are bit-identical to numpy.random.Generator."""
    import numpy
    lib = os.path.join(os.path.dirname(numpy.__file__), "random", "lib", "libnpyrandom.a")
    if not os.path.exists(lib):
        raise RuntimeError(f"{lib} not found (needed by csrc/host_rng.cu)")
    return [lib, "-lm"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build():
    if not os.path.exists(LIB_PATH):
        return True
    lib_mtime = os.path.getmtime(LIB_PATH)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(PKG_DIR, "..", "include", "*.h"))
    return any(os.path.getmtime(p) > lib_mtime for p in deps)


def build(force=False, verbose=False, jobs=None, defines=(), out=None):
    """Compile every csrc/*.cu to an object (in parallel) and link the .so.

    ``defines`` / ``out`` build a tuning variant (e.g. ``-DVR_PAIR_BLOCK=16``)
    into another file, selected at run time with VR_LIB_PATH."""
    lib_path = out or LIB_PATH
    if not force and not defines and out is None and not needs_build():
        return LIB_PATH
    nvcc = _nvcc()
    objdir = os.path.join(PKG_DIR, "build" if not defines else
                          "build_" + "_".join(x.lstrip("-D").replace("=", "") for x in defines))
    os.makedirs(objdir, exist_ok=True)
    procs = []
    objs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        cmd = [nvcc, *NVCC_FLAGS, *defines, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                            stderr=subprocess.STDOUT, text=True)))
    failed = []
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append((cmd, out))
        elif verbose and out.strip():
            print(out, file=sys.stderr)
    if failed:
        msg = "\n".join(" ".join(c) + "\n" + o for c, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    tmp = lib_path + ".tmp"
    link = [nvcc, "-shared", "--cudart", "static",
            "-gencode", "arch=compute_100a,code=sm_100a", *objs, *_npyrandom(), "-o", tmp]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("link failed:\n" + res.stdout + res.stderr)
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    defs = tuple(a for a in sys.argv[1:] if a.startswith("-D"))
    outs = [a[len("--out="):] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose=True, defines=defs,
                out=outs[0] if outs else None))
