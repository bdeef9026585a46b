"""Builds libb2md.so (all CUDA kernels + the C ABI) for sm_100a with nvcc.

In-tree output (``paper_2406_04210_b200/lib/libb2md.so``) so that the built
library travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libb2md.so")

SOURCES = ["state.cu", "cells.cu", "nlist.cu", "force.cu", "integrate.cu",
           "reduce.cu", "sort.cu", "halo.cu", "thermostat.cu", "runtime.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-fvisibility=hidden",
    "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; cannot build libb2md.so")


def sources():
    return [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def is_stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    built = os.path.getmtime(LIB_PATH)
    deps = sources() + [os.path.join(CSRC, "common.cuh"), os.path.join(CSRC, "integrate.cuh"),
                        os.path.join(HERE, "..", "include", "b2md.h")]
    return any(os.path.getmtime(d) > built for d in deps if os.path.exists(d))


def _compile_one(args):
    nvcc, flags, src, obj, verbose = args
    cmd = [nvcc] + flags + (["-Xptxas", "-v"] if verbose else []) + ["-c", "-o", obj, src]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    return src, proc.returncode, proc.stdout + proc.stderr


def build_library(force: bool = False, verbose: bool = False) -> str:
    """One object per translation unit, compiled in parallel (only the stale ones unless
    `force`), then linked into the shared library."""
    if not force and not is_stale():
        return LIB_PATH
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(LIB_DIR, exist_ok=True)
    obj_dir = os.path.join(LIB_DIR, "obj")
    os.makedirs(obj_dir, exist_ok=True)
    extra = os.environ.get("B2MD_NVCC_EXTRA", "").split()      # experiments (-D...)
    nvcc = _nvcc()
    flags = [f for f in NVCC_FLAGS if f != "-shared"] + extra
    headers = [os.path.join(CSRC, "common.cuh"), os.path.join(CSRC, "integrate.cuh"),
               os.path.join(HERE, "..", "include", "b2md.h")]
    newest_header = max(os.path.getmtime(h) for h in headers if os.path.exists(h))
    stamp = os.path.join(obj_dir, "flags.txt")
    flag_text = " ".join(flags)
    same_flags = os.path.exists(stamp) and open(stamp).read() == flag_text
    jobs, objs = [], []
    for src in sources():
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        fresh = (not force and same_flags and os.path.exists(obj) and
                 os.path.getmtime(obj) > max(os.path.getmtime(src), newest_header))
        if not fresh or verbose:
            jobs.append((nvcc, flags, src, obj, verbose))
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4) or 1) as pool:
        results = list(pool.map(_compile_one, jobs))
    failed = [(s, out) for s, rc, out in results if rc != 0]
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(f"{s}:\n{out}" for s, out in failed))
    with open(stamp, "w") as fh:
        fh.write(flag_text)
    if verbose:
        for s, _, out in results:
            print(out)
    proc = subprocess.run([nvcc, "-shared", "-o", LIB_PATH] + objs, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError("link failed:\n" + proc.stdout + proc.stderr)
    return LIB_PATH


if __name__ == "__main__":
    print(build_library(force=True, verbose=True))
