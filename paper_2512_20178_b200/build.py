"""Build libshiro.so in-tree: nvcc for sm_100a kernels, g++ for the host
planner/runtime, NCCL from the torch wheel (nvidia-nccl, 2.28.x).

    python -m paper_2512_20178_b200.build [--force]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libshiro.so")
BUILD = os.path.join(HERE, "build")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    import nvidia.nccl as m   # torch's bundled NCCL (same soname torch loads)
    base = list(m.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "shiro.h")]
    if not force and os.path.exists(OUT):
        t = os.path.getmtime(OUT)
        if all(os.path.getmtime(d) <= t for d in deps):
            return OUT
    os.makedirs(BUILD, exist_ok=True)
    inc, lib = nccl_paths()
    common = ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc]
    jobs = []
    objs = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        if s.endswith(".cu"):
            cmd = [os.path.join(CUDA, "bin", "nvcc"), *ARCH, "-O3", "-lineinfo", "-std=c++17",
                   "-Xptxas", "-v", "-Xcompiler", "-fPIC", *common, "-c", s, "-o", o]
        else:
            cmd = ["g++", "-O2", "-g", "-std=c++17", "-fPIC", "-Wall", "-Wno-unused-function",
                   "-I", os.path.join(CUDA, "include"), *common, "-c", s, "-o", o]
        jobs.append(cmd)
    with ThreadPoolExecutor(max_workers=8) as ex:
        logs = list(ex.map(_run, jobs))
    if verbose:
        print("\n".join(logs))
    with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    link = [os.path.join(CUDA, "bin", "nvcc"), *ARCH, "-shared", "-o", OUT + ".tmp", *objs,
            "-cudart", "static", "-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib,
            "-lpthread"]
    _run(link)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
