"""Build the native library in-tree: nvcc for sm_100a, one shared object.

`python -m paper_2006_06762_b200.build` (or `__graft_entry__.build()`) writes
`paper_2006_06762_b200/_lib/libloomtune_b200.so` plus the NVRTC compile worker
`paper_2006_06762_b200/_lib/lt_nvrtc_worker` and the native State encoder
`paper_2006_06762_b200/_lib/_lt_encode*.so` (CPython extension, g++).  Objects are rebuilt only when a
source is newer than its output.
"""

from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(LIBDIR, "libloomtune_b200.so")
WORKER = os.path.join(LIBDIR, "lt_nvrtc_worker")
ENCODER = os.path.join(LIBDIR, "_lt_encode" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

# exact-arithmetic kernels must not contract a*b+c into an FMA
SOURCES = {
    "features.cu": ["--fmad=false"],
    "predict.cu": ["--fmad=false"],
    "gbdt.cu": ["--fmad=false"],
    "api.cu": [],
    "runner.cu": [],
    "comm.cu": [],
    "compile_pool.cpp": [],
}


def _stale(out: str, deps: list) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def build(verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".h")] + \
        [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE) if f.endswith(".h")]
    objs = []
    for src, extra in SOURCES.items():
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(LIBDIR, src.rsplit(".", 1)[0] + ".o")
        objs.append(obj)
        if _stale(obj, [path] + headers + [__file__]):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-I", CSRC, "-I", INCLUDE, "-I", os.path.join(CUDA, "include"), *extra, "-c", path, "-o", obj]
            if src.endswith(".cpp"):
                cmd = [NVCC, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", CSRC, *extra, "-c", path, "-o", obj]
            if verbose:
                print(" ".join(cmd))
            _run(cmd)
    if _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-ldl",
              "-Xlinker", "-rpath=" + os.path.join(CUDA, "lib64")])
    wsrc = os.path.join(CSRC, "nvrtc_worker.cpp")
    if os.path.exists(wsrc) and _stale(WORKER, [wsrc] + headers):
        _run(["g++", "-O2", "-std=c++17", "-I", os.path.join(CUDA, "include"), wsrc, "-o", WORKER,
              "-L", os.path.join(CUDA, "lib64"), "-lnvrtc", "-lnvptxcompiler_static", "-lpthread", "-lm",
              "-Wl,-rpath," + os.path.join(CUDA, "lib64")])
    esrc = os.path.join(CSRC, "encode_ext.cpp")
    if os.path.exists(esrc) and _stale(ENCODER, [esrc, __file__]):
        _run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-fvisibility=hidden",
              "-I", sysconfig.get_paths()["include"], esrc, "-o", ENCODER])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
