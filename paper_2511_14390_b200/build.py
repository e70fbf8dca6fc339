"""Build libiirgrad.so (sm_100a) in-tree with nvcc.

    python -m paper_2511_14390_b200.build [--force] [--verbose]

Every translation unit under csrc/ is compiled in parallel with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into
``paper_2511_14390_b200/lib/libiirgrad.so``.  Objects are rebuilt only when a
source or header is newer than them.
"""
from __future__ import annotations

import argparse
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# Experiment variants (never the default build): IIRG_VARIANT=name IIRG_DEFS="-DX=1 ..."
# builds build_<name>/ and lib/libiirgrad_<name>.so; load one with IIRG_LIB=<path>.
VARIANT = os.environ.get("IIRG_VARIANT", "")
DEFS = os.environ.get("IIRG_DEFS", "").split() if VARIANT else []
BUILD = os.path.join(HERE, "build" + (f"_{VARIANT}" if VARIANT else ""))
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libiirgrad" + (f"_{VARIANT}" if VARIANT else "") + ".so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
                f"-I{INCLUDE}", "--expt-relaxed-constexpr"]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))


def _deps(obj, fallback):
    """Headers an object depends on, from the nvcc -MD file of its last compile (all
    headers when there is none)."""
    try:
        txt = open(obj + ".d").read().replace("\\\n", " ")
    except OSError:
        return fallback
    deps = [d for d in txt.split(":", 1)[1].split() if d.startswith(CSRC) or d.startswith(INCLUDE)]
    return [d for d in deps if os.path.exists(d)] or fallback


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = _headers()
    objs = []
    todo = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + _deps(o, hdrs)):
            todo.append((s, o))

    def compile_one(so):
        s, o = so
        cmd = [NVCC] + FLAGS + DEFS + (["-Xptxas", "-v"] if verbose else []) + \
            ["-MD", "-MF", o + ".d", "-c", s, "-o", o + ".tmp"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{r.stdout}\n{r.stderr}")
        os.replace(o + ".tmp", o)
        return s, r.stderr

    if todo:
        with ThreadPoolExecutor(jobs or min(len(todo), os.cpu_count() or 4)) as ex:
            for s, err in ex.map(compile_one, todo):
                if verbose and err:
                    print(f"== {os.path.basename(s)}\n{err}", file=sys.stderr)
    if force or todo or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart"]
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
