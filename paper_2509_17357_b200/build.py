"""In-tree build of libcronus_b200.so (host C++ scheduler + GPU engine + sm_100a kernels).

    python -m paper_2509_17357_b200.build [-j N] [--clean]

Host C++ is compiled with g++ (-ffp-contract=off: the virtual clock must round
exactly like the oracle), CUDA with nvcc for sm_100a only. The CUDA runtime is
linked statically so the library loads on a CPU-only machine (virtual-clock entry
points work there) and on the GPU box without a toolkit path. Incremental: an
object is rebuilt when its source or any header is newer.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libcronus_b200.so")
CLI = os.path.join(PKG, "cronus_b200")  # command-line driver (csrc/cli)
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def json_include() -> str:
    for d in sys.path + [sysconfig.get_paths()["purelib"]]:
        p = os.path.join(d, "include", "cudnn_frontend", "thirdparty", "nlohmann")
        if os.path.exists(os.path.join(p, "json.hpp")):
            return p
    raise RuntimeError("nlohmann/json.hpp not found (expected under site-packages/include/cudnn_frontend)")


def includes() -> list[str]:
    return ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-I" + json_include(),
            "-I" + os.path.join(CUDA, "include")]


def sources():
    host = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    gpu_cpp = sorted(glob.glob(os.path.join(CSRC, "gpu", "*.cpp")))
    cu = sorted(glob.glob(os.path.join(CSRC, "kernels", "*.cu")) + glob.glob(os.path.join(CSRC, "gpu", "*.cu")))
    return host + gpu_cpp, cu


def headers_mtime() -> float:
    hs = glob.glob(os.path.join(CSRC, "**", "*.h*"), recursive=True)
    hs += glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
    hs += glob.glob(os.path.join(ROOT, "include", "**", "*.h*"), recursive=True)
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def obj_for(src: str) -> str:
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(BUILD, rel + ".o")


def compile_cmd(src: str, obj: str) -> list[str]:
    if src.endswith(".cu"):
        return [NVCC, "-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC",
                "--expt-relaxed-constexpr", "-Xptxas", "-v", *includes(), "-c", src, "-o", obj]
    return [CXX, "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall", "-Wno-unused-function",
            *includes(), "-c", src, "-o", obj]


def build(jobs: int | None = None, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    cpp, cu = sources()
    hdr = headers_mtime()
    todo = []
    for s in cpp + cu:
        o = obj_for(s)
        if not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr):
            todo.append((s, o))

    def run(item):
        s, o = item
        cmd = compile_cmd(s, o)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {os.path.relpath(s, ROOT)}\n{r.stdout}\n{r.stderr}")
        if s.endswith(".cu"):
            with open(o + ".ptxas.txt", "w") as f:
                f.write(r.stderr)
        return s

    if todo:
        with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
            for s in ex.map(run, todo):
                if verbose:
                    print("compiled", os.path.relpath(s, ROOT))
    objs = [obj_for(s) for s in cpp + cu]
    if todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        # no device-link step: relocatable device code is not used (static cudart)
        cmd = [CXX, "-shared", "-o", LIB, *objs, "-L" + os.path.join(CUDA, "lib64"),
               "-lcudart_static", "-lrt", "-lpthread", "-ldl", "-Wl,--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
        if verbose:
            print("linked", os.path.relpath(LIB, ROOT))
    # the command-line driver (cronus_sim's subcommands), linked against the library
    cli_src = os.path.join(CSRC, "cli", "cronus_b200.cpp")
    if not os.path.exists(CLI) or os.path.getmtime(CLI) < max(os.path.getmtime(cli_src), os.path.getmtime(LIB), hdr):
        cmd = [CXX, "-std=c++20", "-O2", *includes(), cli_src, "-o", CLI, "-L" + PKG, "-lcronus_b200",
               "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"cli build failed\n{r.stdout}\n{r.stderr}")
        if verbose:
            print("linked", os.path.relpath(CLI, ROOT))
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("--clean", action="store_true")
    a = ap.parse_args()
    if a.clean and os.path.exists(BUILD):
        shutil.rmtree(BUILD)
    print(build(a.j, verbose=True))


if __name__ == "__main__":
    main()
