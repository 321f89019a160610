"""Build libvecflow.so in-tree for sm_100a (nvcc; no JIT, no torch extension machinery)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libvecflow.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU = ["route.cu", "scan.cu", "scan_tc.cu", "graph_build.cu", "graph.cu", "merge.cu", "small.cu"]
CPP = ["vf_api.cpp", "shard.cpp", "serve.cpp"]
HEADERS = ["vf_internal.h", "common.cuh", "tc_common.cuh", "host_internal.h", "graph_item.cuh", "small.h"]


def _sources():
    return [os.path.join(CSRC, f) for f in CU + CPP + HEADERS] + [os.path.join(ROOT, "include", "vf.h")]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(s) <= t for s in _sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
              "-I" + CSRC]
    common += os.environ.get("VF_NVCC_EXTRA", "").split()      # e.g. -DVF_TC_PROF (diagnostics builds)
    def compile_one(f):
        src = os.path.join(CSRC, f)
        obj = os.path.join(objdir, f + ".o")
        cmd = [NVCC] + ARCH + common + ["--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
                                         "-c", src, "-o", obj]
        if f.endswith(".cpp"):
            cmd = [NVCC] + common + ["-x", "c++", "-c", src, "-o", obj]
        return f, obj, subprocess.run(cmd, capture_output=True, text=True)

    # translation units compile in parallel (nvcc is single-threaded per file)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(CU + CPP), os.cpu_count() or 1)) as ex:
        done = list(ex.map(compile_one, CU + CPP))
    objs = []
    for f, obj, r in done:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed for {f}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    tmp = OUT + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs + ["-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="-f" in sys.argv, verbose="-v" in sys.argv))
