"""In-tree build of libamg_b200.so (host setup in C++/OpenMP, solve kernels in CUDA for sm_100a).

    python -m paper_2511_21268_b200.build [--force] [--verbose] [--checked]

Host files are compiled with -ffp-contract=off (the canonical arithmetic contract of DESIGN.md §3:
no FMA contraction in the generator or the setup).  Device code is compiled for sm_100a only.
"""
from __future__ import annotations

import concurrent.futures
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libamg_b200.so")
# checked build: device-side invariant checks (AMG_CHECKS in kernels.cuh), loaded with AMG_LIB=checked
BUILD_CHECKED = os.path.join(HERE, "_build_checked")
LIB_CHECKED = os.path.join(HERE, "libamg_b200_checked.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")

HOST_SRCS = ["api.cpp", "iga_gen.cpp", "setup.cpp", "dist.cpp", "share.cpp"]
CUDA_SRCS = ["device.cu", "inst_cheb.cu", "inst_cheb_dot.cu", "inst_spmv.cu", "inst_transfer.cu",
             "inst_vi_cheb.cu", "inst_vi_cheb_dot.cu", "inst_vi_spmv.cu", "inst_vi_transfer.cu"]
HEADERS = ["common.hpp", "kernels.cuh", "devstate.cuh", "launch_csr.cuh", "launch_csr_vi.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    build_dir, lib_out = (BUILD_CHECKED, LIB_CHECKED) if checked else (BUILD, LIB)
    os.makedirs(build_dir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "amg_b200.h")]
    jobs, objs = [], []
    for src in HOST_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            jobs.append(["g++", "-O2", "-std=gnu++17", "-fPIC", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
                         "-Wall", "-Wno-unknown-pragmas", "-I", INCLUDE, "-c", s, "-o", o])
    for src in CUDA_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v", "--expt-relaxed-constexpr",
                         *(["-DAMG_CHECKS"] if checked else []),
                         "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off", "-I", INCLUDE, "-c", s, "-o", o])
    # the translation units are independent: compile them in parallel
    with concurrent.futures.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(_run, j, verbose) for j in jobs]:
            f.result()
    if force or _newer(lib_out, objs):
        tmp = lib_out + f".tmp{os.getpid()}"
        _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fopenmp", "-Xlinker", "--no-undefined",
              "-lgomp", "-lquadmath", "-lnccl", "-lcudart"], verbose)
        os.replace(tmp, lib_out)
    return lib_out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, checked="--checked" in sys.argv))
