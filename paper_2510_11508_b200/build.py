"""Build the in-tree sm_100a shared library ``libnormint_b200.so``.

    python -m paper_2510_11508_b200.build [--force] [--verbose]

Every ``csrc/*.cu`` is compiled by nvcc for ``-gencode
arch=compute_100a,code=sm_100a`` with ``-lineinfo`` (so ncu's source page
maps to the code) and linked with the static CUDA runtime into one C-ABI
library next to this file.  The library exports exactly the functions
declared in ``include/normint_b200.h``.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libnormint_b200.so")
OBJ = os.path.join(ROOT, "build", "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-O3", "-I", os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(ROOT, "include", "normint_b200.h")]


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    return os.path.getmtime(OUT) >= _newest(sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Build the library; ``defines``/``out`` build an experiment variant elsewhere."""
    if out is None and not defines and not force and up_to_date():
        return OUT
    variant = bool(defines) or out is not None
    objdir = OBJ + ("_" + "_".join(d.replace("=", "") for d in defines) if defines else "")
    out = out or OUT
    os.makedirs(objdir, exist_ok=True)
    cc = nvcc()
    hdr_time = _newest(headers() + [__file__])

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        if (not force and not variant and os.path.exists(obj)
                and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_time)):
            return obj
        cmd = [cc, *ARCH, *FLAGS, *(f"-D{d}" for d in defines), "-c", src, "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = out + ".tmp"
    cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, out)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("-D", dest="defines", action="append", default=[],
                    help="extra preprocessor define (experiment variants; needs --out)")
    ap.add_argument("--out", default=None, help="output path for a variant build")
    a = ap.parse_args()
    print(build(a.force, a.verbose, tuple(a.defines), a.out))


if __name__ == "__main__":
    main()
