"""Builds libl0search.so in-tree with nvcc for sm_100a (no torch, no JIT cache).

    python -m paper_2502_20072_b200.build [--force] [-j N]

Each translation unit in csrc/ is compiled separately (in parallel) and the
objects are linked into one shared library with the CUDA runtime linked
statically, so the .so that travels to the GPU box has no build-time
dependencies.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "csrc", "_obj")
LIB = os.path.join(HERE, "libl0search.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
              "-Xptxas", "-v", f"-I{INCLUDE}"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _deps_mtime() -> float:
    paths = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    paths.append(os.path.join(INCLUDE, "l0search.h"))
    return max(os.path.getmtime(p) for p in paths)


def _compile(src: str, objdir: str = OBJ, defines: tuple = ()) -> tuple[str, str]:
    obj = os.path.join(objdir, os.path.splitext(os.path.basename(src))[0] + ".o")
    if src.endswith(".cpp"):  # host-only code (intrinsics): the host compiler directly
        cmd = ["g++", "-O3", "-fPIC", "-std=c++17", f"-I{INCLUDE}", *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
    else:
        cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, jobs: int | None = None, verbose: bool = False, defines: tuple = (),
          out: str | None = None) -> str:
    """Build the library; `defines`/`out` produce a tuning variant (e.g. L0S_CFG34=...)."""
    lib_path = out or LIB
    if not force and os.path.exists(lib_path) and os.path.getmtime(lib_path) >= _deps_mtime():
        return lib_path
    # tuning variants compile in a scratch directory outside the tree (removed after linking)
    objdir = OBJ if not defines else tempfile.mkdtemp(prefix="l0s_variant_obj_")
    os.makedirs(objdir, exist_ok=True)
    srcs = sources()
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(lambda s: _compile(s, objdir, defines), srcs))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    objs = [o for o, _ in results]
    LIB_OUT = lib_path
    tmp = LIB_OUT + ".tmp"
    r = subprocess.run([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-lpthread", "-ldl"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB_OUT)
    if defines:
        shutil.rmtree(objdir, ignore_errors=True)
        return LIB_OUT
    with open(os.path.join(objdir, "ptxas.log"), "w") as fh:
        for _, log in results:
            fh.write(log)
    return LIB_OUT


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("-v", action="store_true")
    args = ap.parse_args()
    print(build(force=args.force, jobs=args.j, verbose=args.v))


if __name__ == "__main__":
    main()
