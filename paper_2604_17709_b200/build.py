"""Build the C-ABI library in-tree with nvcc for sm_100a.

    python -m paper_2604_17709_b200.build [--force]

Each csrc/*.cu is compiled with
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17
and linked (static cudart) into two libraries:
    libdl.so     the release library: behaviour fixed by include/dl.h alone
    libdl_ab.so  the same sources with -DDL_AB_SWITCHES: the measured-and-lost
                 design alternatives become selectable by environment variable
                 (A/B switches) for re-measurement and their parity
                 tests; selected by DL_LIBRARY=ab (paper_2604_17709_b200/_lib.py)
Objects are cached under paper_2604_17709_b200/build{,_ab}/ and rebuilt when a
source or header is newer.  Compiles run in parallel.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
VARIANTS = {"release": (os.path.join(HERE, "build"), os.path.join(HERE, "libdl.so"), []),
            "ab": (os.path.join(HERE, "build_ab"), os.path.join(HERE, "libdl_ab.so"), ["-DDL_AB_SWITCHES"])}
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


def _compile(src: str, force: bool, obj_dir: str, extra) -> str:
    obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
    newest = max([os.path.getmtime(src)] + [os.path.getmtime(h) for h in _headers()])
    if force or not os.path.exists(obj) or os.path.getmtime(obj) < newest:
        cmd = [NVCC] + ARCH + FLAGS + extra + ["-c", src, "-o", obj + ".tmp"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        os.replace(obj + ".tmp", obj)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    """Build both variants; returns the release library's path."""
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = [(s, v) for v in VARIANTS for s in srcs]
    for obj_dir, _, _ in VARIANTS.values():
        os.makedirs(obj_dir, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=8) as ex:
        objs = list(ex.map(lambda j: _compile(j[0], force, VARIANTS[j[1]][0], VARIANTS[j[1]][2]), jobs))
    for v, (obj_dir, lib, _) in VARIANTS.items():
        _link([o for o, j in zip(objs, jobs) if j[1] == v], lib, force)
    if verbose:
        print(VARIANTS["release"][1])
    return VARIANTS["release"][1]


def _link(objs, LIB: str, force: bool) -> None:
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
