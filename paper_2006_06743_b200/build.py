"""Build libsngb.so (the C-ABI library) in-tree for sm_100a.

    python -m paper_2006_06743_b200.build [--verbose]
    python -m paper_2006_06743_b200.build --variant NAME -DMACRO=1 ...   (A/B builds)

A variant compiles with the extra nvcc flags into build/NAME/ and links
tools/ab/libsngb_NAME.so (select it at run time with SNGB_LIBRARY=...).

Objects are compiled in parallel with nvcc and linked into
paper_2006_06743_b200/lib/libsngb.so, which travels to the GPU box with the
repo snapshot (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "lib", "libsngb.so")
CLI_SRC = os.path.join(PKG, "cpp", "tools", "sngb_cluster.cpp")
CLI = os.path.join(PKG, "bin", "sngb_cluster")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["sngb_api.cu", "sngb_kernels.cu", "sngb_quant.cu", "sngb_metric.cu", "sngb_head.cu", "sngb_sampler.cu",
           "sngb_cluster.cu", "sngb_multi.cu", "sngb_fused.cu"]
HEADERS = ["sngb_internal.cuh", "sngb_host.cuh", "sngb_rng.cuh", "sngb_device.cuh", "sngb_epstest.cuh",
           "sngb_floyd_bitmap.cuh", "sngb_floyd_bloom.cuh", "sngb_floyd_warp.cuh", "sngb_floyd_lean.cuh", "sngb_floyd_pipe.cuh", "sngb_floyd_headpipe.cuh", "sngb_floyd_head.cuh",
           "sngb_head.cuh", "sngb_gather_head.cuh"]

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "-I" + os.path.join(ROOT, "include"),
    "-I" + CSRC,
]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool, obj_dir: str = OBJ, extra: tuple = ()) -> str:
    obj = os.path.join(obj_dir, os.path.splitext(src)[0] + ".o")
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + \
        [os.path.join(ROOT, "include", "sngb.h")]
    if _stale(obj, deps):
        cmd = [NVCC, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return obj


def build(verbose: bool = False, variant: str | None = None, extra: tuple = ()) -> str:
    obj_dir = os.path.join(OBJ, variant) if variant else OBJ
    lib = os.path.join(ROOT, "tools", "ab", f"libsngb_{variant}.so") if variant else LIB
    os.makedirs(obj_dir, exist_ok=True)
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    if variant:  # always rebuild: the flags are not part of the staleness check
        for src in SOURCES:
            o = os.path.join(obj_dir, os.path.splitext(src)[0] + ".o")
            if os.path.exists(o):
                os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, obj_dir, tuple(extra)), SOURCES))
    if variant or _stale(lib, objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs,
               "-lcudart", "-lpthread"]
        subprocess.run(cmd, check=True)
    if not variant:
        build_testhooks(objs)
        build_cli(lib)
        build_pymod(lib)
    return lib


TESTHOOKS_LIB = os.path.join(PKG, "lib", "libsngb_testhooks.so")


def build_testhooks(objs: list[str]) -> str:
    """lib/libsngb_testhooks.so: the product objects with sngb_api.cu recompiled
    with -DSNGB_TEST_HOOKS (SNGB_TEST_FORCE_IRREGULAR forces the exact replay
    path).  Loaded only by tests/conftest.py, never by the package."""
    hook_dir = os.path.join(OBJ, "testhooks")
    os.makedirs(hook_dir, exist_ok=True)
    api = _compile("sngb_api.cu", False, hook_dir, ("-DSNGB_TEST_HOOKS=1",))
    others = [o for o in objs if os.path.basename(o) != "sngb_api.o"]
    if _stale(TESTHOOKS_LIB, [api, *others]):
        subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                        TESTHOOKS_LIB, api, *others, "-lcudart", "-lpthread"], check=True)
    return TESTHOOKS_LIB


PYMOD_SRC = os.path.join(PKG, "cpp", "python", "sngdbscan_module.cpp")
PYMOD_DIR = os.path.join(ROOT, "sngdbscan")


def build_pymod(lib: str = LIB) -> str:
    """The `sngdbscan` pybind11 module (reference proj/CMakeLists.txt:11) ->
    sngdbscan/_sngdbscan<EXT_SUFFIX>, linked against libsngb.so."""
    import sysconfig

    import pybind11

    out = os.path.join(PYMOD_DIR, "_sngdbscan" + sysconfig.get_config_var("EXT_SUFFIX"))
    deps = [PYMOD_SRC, lib, os.path.join(ROOT, "include", "sngb.h")]
    if _stale(out, deps):
        libdir = os.path.dirname(lib)
        rel = os.path.relpath(libdir, PYMOD_DIR)
        subprocess.run([os.environ.get("CXX", "g++"), "-std=c++17", "-O2", "-shared", "-fPIC",
                        "-fvisibility=hidden", "-I" + pybind11.get_include(),
                        "-I" + sysconfig.get_paths()["include"],
                        "-I" + os.path.join(ROOT, "include"), PYMOD_SRC, "-L" + libdir, "-lsngb",
                        f"-Wl,-rpath,$ORIGIN/{rel}", "-o", out], check=True)
    return out


def build_cli(lib: str = LIB) -> str:
    """The `cluster` front-end (SPEC cmd_cluster) over the C++ mirror -> bin/sngb_cluster."""
    inc = os.path.join(PKG, "cpp", "include")
    deps = [CLI_SRC, lib, os.path.join(ROOT, "include", "sngb.h"),
            os.path.join(inc, "sngb", "sng.hpp"), os.path.join(inc, "sngb", "io.hpp")]
    if _stale(CLI, deps):
        os.makedirs(os.path.dirname(CLI), exist_ok=True)
        libdir = os.path.dirname(lib)
        subprocess.run([os.environ.get("CXX", "g++"), "-std=c++20", "-O2", "-Wall",
                        "-I" + os.path.join(ROOT, "include"), "-I" + inc, CLI_SRC,
                        "-L" + libdir, "-lsngb", "-Wl,-rpath,$ORIGIN/../lib", "-o", CLI],
                       check=True)
    return CLI


if __name__ == "__main__":
    argv = sys.argv[1:]
    name = None
    if "--variant" in argv:
        i = argv.index("--variant")
        name = argv[i + 1]
        argv = argv[:i] + argv[i + 2:]
    print(build(verbose="--verbose" in argv, variant=name,
                extra=tuple(a for a in argv if a != "--verbose")))
