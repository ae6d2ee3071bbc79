"""Build libptdr.so in-tree: nvcc for sm_100a only (no other arch, no JIT)."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
TRACE_BUILD = os.environ.get("PTDR_TRACE_BUILD") == "1"  # developer timeline build
# Developer diagnostic builds: PTDR_DIAG_BUILD=<bits> compiles dense_pipe.cuh with
# -DPTDR_DIAG=<bits> into libptdr_diag<bits>.so (never loaded by the product path).
DIAG_BUILD = os.environ.get("PTDR_DIAG_BUILD", "")
# PTDR_DEV_BUILD=1: libptdr_dev.so with every pipeline configuration and the PTDR_*
# environment switches (DESIGN.md section 7 sweeps).  Trace and diagnostic builds are
# developer builds too.  The product library reads no environment variable.
DEV_BUILD = os.environ.get("PTDR_DEV_BUILD") == "1"
_VARIANT = "_trace" if TRACE_BUILD else (f"_diag{DIAG_BUILD}" if DIAG_BUILD else ("_dev" if DEV_BUILD else ""))
IS_DEV = bool(_VARIANT)
# pipeline configurations only developer builds instantiate (dense_plan.h pipe_cfg_built)
DEV_ONLY_SOURCES = {f"dense_pipe_c{k}.cu" for k in (2, 3, 5, 6, 7, 8)}
BUILD = os.path.join(HERE, "_build" + _VARIANT)
LIB = os.path.join(HERE, f"libptdr{_VARIANT}.so")
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    f"-I{os.path.join(ROOT, 'include')}",
] + (["-DPTDR_ENABLE_TRACE=1"] if TRACE_BUILD else []) + ([f"-DPTDR_DIAG={DIAG_BUILD}"] if DIAG_BUILD else []) \
  + (["-DPTDR_DEV=1"] if IS_DEV else [])


def _deps():
    return (glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
            + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "ptdr.h")])


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose):
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
    cmd = [NVCC] + NVCC_FLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = obj + ".log"
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    if verbose:
        print(f"[ptdr build] {os.path.basename(src)}", file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    deps = _deps()
    if not force and not _stale(LIB, deps):
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(s for s in glob.glob(os.path.join(CSRC, "*.cu"))
                  if IS_DEV or os.path.basename(s) not in DEV_ONLY_SOURCES)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp] + objs
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
