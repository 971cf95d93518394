"""In-tree build of libfeod.so for sm_100a (nvcc + g++, no JIT cache).

``python -m paper_2506_00746_b200.build`` or ``__graft_entry__.build()``.
Objects go to ``paper_2506_00746_b200/build/``; the shared library is written
next to this file so it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libfeod.so")
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
           "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _sources():
    cu = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    cpp = sorted(f for f in os.listdir(CSRC) if f.endswith(".cpp"))
    hdr = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hdr.append(os.path.join(ROOT, "include", "feod.h"))
    return cu, cpp, hdr


def _stale(obj, src, hdrs):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src] + hdrs)


def build(verbose: bool = False, jobs: int | None = None, extra: list[str] | None = None,
          lib: str | None = None) -> str:
    """Compile and link libfeod. ``extra`` nvcc flags (experiment variants) build into
    their own object directory (keyed by a hash of the flags) and, unless ``lib`` says
    otherwise, link to abtest/libfeod_<hash>.so -- never over the default build."""
    import hashlib
    build_dir, out_lib = BUILD, LIB
    if extra:
        tag = hashlib.sha1(" ".join(extra).encode()).hexdigest()[:10]
        build_dir = BUILD + "_" + tag
        out_lib = os.path.join(ROOT, "abtest", f"libfeod_{tag}.so")
    if lib:
        out_lib = lib
    os.makedirs(build_dir, exist_ok=True)
    os.makedirs(os.path.dirname(out_lib), exist_ok=True)
    cu, cpp, hdrs = _sources()
    cmds = []
    objs = []
    for f in cu:
        src, obj = os.path.join(CSRC, f), os.path.join(build_dir, f + ".o")
        objs.append(obj)
        if _stale(obj, src, hdrs):
            cmds.append([NVCC, *ARCH, *NVFLAGS, *(extra or []), "-c", src, "-o", obj])
    for f in cpp:
        src, obj = os.path.join(CSRC, f), os.path.join(build_dir, f + ".o")
        objs.append(obj)
        if _stale(obj, src, hdrs):
            cmds.append(["g++", "-O2", "-std=c++17", "-fPIC", "-fvisibility=hidden", "-c", src, "-o", obj])

    def run(cmd):
        res = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, res

    with cf.ThreadPoolExecutor(max_workers=jobs or max(2, os.cpu_count() or 2)) as ex:
        for cmd, res in ex.map(run, cmds):
            if verbose or res.returncode:
                sys.stderr.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            if res.returncode:
                raise RuntimeError(f"compile failed: {cmd[-3]}")
    if cmds or not os.path.exists(out_lib) or any(os.path.getmtime(o) > os.path.getmtime(out_lib) for o in objs):
        link = [NVCC, *ARCH, "-shared", "-o", out_lib, *objs, "-cudart", "static", "-Xcompiler", "-fPIC"]
        res = subprocess.run(link, capture_output=True, text=True)
        if verbose or res.returncode:
            sys.stderr.write(" ".join(link) + "\n" + res.stdout + res.stderr)
        if res.returncode:
            raise RuntimeError("link failed")
    return out_lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
