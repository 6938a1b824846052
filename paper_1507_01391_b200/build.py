"""Build libdmm_b200.so in-tree: every csrc/*.cu compiled for sm_100a in parallel, then
linked into one shared library (the C ABI of include/dmm_gpu.h).

    python -m paper_1507_01391_b200.build [-v] [-j N]

nvcc cross-compiles without a GPU; the .so travels to the GPU box with the repo.
Objects are rebuilt only when a source or any header under csrc/ or include/ is newer.
"""
from __future__ import annotations

import argparse
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libdmm_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2",
         "-I" + os.path.join(ROOT, "include")]


def _headers() -> list[str]:
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(CSRC, "*.inc")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool, obj_dir: str = OBJ, defines: tuple = ()) -> tuple[str, str]:
    obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
    if not _stale(obj, [src] + _headers()):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stdout + r.stderr


def build(verbose: bool = False, jobs: int = 0, defines: tuple = (), out: str = "") -> str:
    """Build the library; `defines` + `out` build a diagnostic variant (e.g. DMM_NO_GLOBAL_IO into
    paper_1507_01391_b200/_variants/) with its own object directory."""
    obj_dir, lib_path = OBJ, LIB
    if defines:
        tag = "_".join(d.replace("=", "_").lower() for d in defines)
        obj_dir = os.path.join(PKG, "_build_" + tag)
        lib_path = out or os.path.join(PKG, "_variants", f"libdmm_b200_{tag}.so")
        os.makedirs(os.path.dirname(lib_path), exist_ok=True)
    os.makedirs(obj_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose, obj_dir, tuple(defines)), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for (_, log), s in zip(results, srcs):
            if log:
                print(f"== {os.path.basename(s)}\n{log}")
    if _stale(lib_path, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib_path, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib_path


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("-j", "--jobs", type=int, default=0)
    ap.add_argument("-D", "--define", action="append", default=[], help="diagnostic variant macro")
    a = ap.parse_args()
    print(build(a.verbose, a.jobs, tuple(a.define)))


if __name__ == "__main__":
    sys.exit(main())
