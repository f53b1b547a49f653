"""Build the in-tree CUDA library ``_lib/libgrkan_b200.so`` for sm_100a.

    python -m paper_2505_13813_b200.build [--force] [--ptxas-v]

One nvcc process per translation unit (host C ABI + one kernel TU per I/O
dtype), run in parallel, then one shared-library link.  nvcc cross-compiles
without a GPU; the .so is git-ignored but travels to the GPU box with the repo.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib", "libgrkan_b200.so")
OBJ_DIR = os.path.join(HERE, "_lib", "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler",
              "-fvisibility=hidden", "-I", os.path.join(ROOT, "include")] + ARCH


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "grkan_b200.h"), os.path.abspath(__file__)]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = True, ptxas_v: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile the library.  ``out`` / ``defines`` make tuning variants (tools/build_variant.py)."""
    target = out or OUT
    if not force and out is None and up_to_date():
        return OUT
    obj_dir = OBJ_DIR if out is None else os.path.join(os.path.dirname(target), "obj")
    os.makedirs(obj_dir, exist_ok=True)
    cc = nvcc()
    extra = (["-Xptxas", "-v"] if ptxas_v else []) + ["-D%s" % d for d in defines]

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        cmd = [cc] + NVCC_FLAGS + extra + ["-c", "-o", obj, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s" % (src, r.stderr))
        return obj, r.stderr

    with ThreadPoolExecutor(max_workers=len(sources())) as pool:
        results = list(pool.map(compile_one, sources()))
    if ptxas_v:
        with open(os.path.join(obj_dir, "ptxas.log"), "w") as fh:
            for _, log in results:
                fh.write(log)
    tmp = target + ".tmp"
    cmd = [cc] + ARCH + ["-shared", "-o", tmp] + [o for o, _ in results]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, ptxas_v="--ptxas-v" in sys.argv)
