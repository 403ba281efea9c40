"""Build libsvdsb.so in-tree with nvcc for sm_100a.

    python -m paper_1607_01404_b200.build [--force] [--verbose]

The shared library lands next to this file (``_lib/libsvdsb.so``) so it
travels with the repository snapshot to the GPU box; nothing is installed
into site-packages and no JIT cache is used.
"""

import argparse
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libsvdsb.so")
REPO = os.path.dirname(HERE)

SOURCES = ["runtime.cu", "csr.cu", "dense.cu", "small.cu", "arrow.cu", "jdqmr.cu", "gdk.cu", "mmio.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _inputs():
    files = [os.path.join(CSRC, s) for s in SOURCES]
    files += [os.path.join(CSRC, f) for f in os.listdir(CSRC)
              if f.endswith((".cuh", ".h"))]
    files.append(os.path.join(REPO, "include", "svdsb.h"))
    return files


STAMP = LIB + ".srchash"


def source_hash():
    """SHA-256 over the compiler version, flags and every input file's
    contents: the library is reused only when it was built from exactly
    these sources (file times say nothing after a checkout or a copy)."""
    import hashlib
    h = hashlib.sha256()
    try:
        h.update(subprocess.run([NVCC, "--version"], capture_output=True).stdout)
    except OSError:
        pass
    h.update(" ".join(ARCH + FLAGS).encode())
    for f in sorted(_inputs()):
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def up_to_date():
    if not (os.path.exists(LIB) and os.path.exists(STAMP)):
        return False
    with open(STAMP) as fh:
        return fh.read().strip() == source_hash()


def build(force=False, verbose=False, variant=None, overrides=None, defines=()):
    """Compile every .cu to an object, then link the shared library.

    variant / overrides (kernel experiments only): link
    _lib/libsvdsb_<variant>.so with some sources replaced by other files
    (overrides: {"dense.cu": "/path/to/dense.cu"}); loaded when
    SVDSB_LIB_VARIANT=<variant> is set."""
    overrides = overrides or {}
    lib = LIB if variant is None else os.path.join(OUT_DIR, "libsvdsb_%s.so" % variant)
    if variant is None and not force and up_to_date():
        return LIB
    odir = OUT_DIR if variant is None else os.path.join(OUT_DIR, "var_" + variant)
    os.makedirs(odir, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(odir, os.path.splitext(src)[0] + ".o")
        path = overrides.get(src, os.path.join(CSRC, src))
        cmd = [NVCC, *ARCH, *FLAGS, *["-D" + d for d in defines], "-I", os.path.join(REPO, "include"), "-I", CSRC,
               "-c", path, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed on %s" % src)
        if verbose:
            sys.stderr.write(res.stderr)
        objs.append(obj)
    cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    if variant is None and not overrides and not defines:
        with open(STAMP, "w") as fh:
            fh.write(source_hash() + "\n")
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--variant", default=None)
    ap.add_argument("--override", action="append", default=[], metavar="SRC=PATH")
    ap.add_argument("--define", action="append", default=[], metavar="NAME=VALUE")
    args = ap.parse_args()
    ov = dict(o.split("=", 1) for o in args.override)
    print(build(force=args.force, verbose=args.verbose, variant=args.variant, overrides=ov, defines=args.define))


if __name__ == "__main__":
    main()
