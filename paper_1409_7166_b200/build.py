"""Build the sm_100a shared library libpgb200.so in-tree with nvcc.

    python -m paper_1409_7166_b200.build          (or __graft_entry__.build())
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libpgb200.so")
# debugging variant with cycle instrumentation of the sweep kernel (-DPG_PROF)
PROF_LIB = os.path.join(LIBDIR, "libpgb200_prof.so")
SOURCES = ["pg_sweep_fused_i1.cu", "pg_sweep_fused_i2.cu", "pg_sweep_fused_i3.cu", "pg_sweep_fused_i4.cu",
           "pg_sweep_fused_i5.cu", "pg_sweep2.cu", "pg_kernels.cu", "pg_sweep_fused.cu", "pg_api.cu", "pg_group.cu", "pg_store.cu",
           "pg_csr_build.cpp", "pg_csr_device.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "pgrid.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, prof: bool = False, variant: str = "",
          defs: tuple = ()) -> str:
    """prof: the cycle-instrumented library; variant: an experiment library
    lib/libpgb200_<variant>.so compiled with the extra -D flags `defs` (A/B
    runs select it with PGB200_LIB); the default library takes neither."""
    lib = PROF_LIB if prof else (os.path.join(LIBDIR, f"libpgb200_{variant}.so") if variant else LIB)
    if not force and not prof and not variant and not _stale():
        return LIB
    # experiments: extra -D flags for the instrumented build only
    extra = (["-DPG_PROF"] + os.environ.get("PG_EXTRA_DEFS", "").split()) if prof else []
    extra += [f"-D{d}" for d in defs]
    tag = "_prof" if prof else (f"_{variant}" if variant else "")
    os.makedirs(LIBDIR, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(LIBDIR, src.rsplit(".", 1)[0] + tag + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    # translation units compile in parallel (the fused-sweep instances dominate)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    objs = []
    for src, obj, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed for {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, prof="--prof" in sys.argv))
