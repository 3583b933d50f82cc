"""Builds the native libraries in-tree (they travel to the GPU box with the repo snapshot).

  libkernid_cuda.so  -- sm_100a kernels + the C-ABI of include/kernid_cuda.h (nvcc)
  libkernid_host.so  -- the host-side C++ mirror of the reference `kernid::` API
                        (include/kernid_b200.hpp) over the C-ABI (g++, -ffp-contract=off)
"""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
CUDA_SO = os.path.join(PKG, "libkernid_cuda.so")
HOST_SO = os.path.join(PKG, "libkernid_host.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SRCS = ["kid_capi.cu", "kid_split.cu", "kid_passes.cu", "kid_next.cu", "kid_fused.cu", "kid_fused_w.cu", "kid_gram2.cu"]
HOST_SRCS = ["kernid_host.cpp", "kernid_multi.cpp"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(p) > t for p in deps)


def build_cuda(force=False, verbose=False):
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "kernid_cuda.h")]
    if not force and not _stale(CUDA_SO, deps):
        return CUDA_SO
    # one nvcc per translation unit, in parallel (the cluster kernels' template instances dominate)
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, f[:-3] + ".o") for f in CU_SRCS]

    def cc(i):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-c",
               "-Xptxas", "-warn-spills", "-o", objs[i], os.path.join(CSRC, CU_SRCS[i])]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(len(CU_SRCS)) as ex:
        list(ex.map(cc, range(len(CU_SRCS))))
    cmd = [NVCC, *ARCH, "-shared", "-o", CUDA_SO] + objs
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return CUDA_SO


def build_guard(verbose=False):
    """libkernid_cuda_guard.so: the same objects with kid_capi.cu compiled -DKID_GUARD (64 KB canary zones
    around every device buffer, kid_guard_check) -- the out-of-bounds check of tools/guard_cases.py, built on
    demand (compute-sanitizer is closed on this GPU pool). Not part of build_all."""
    build_cuda(False, verbose)
    objdir = os.path.join(PKG, "build")
    gobj = os.path.join(objdir, "kid_capi_guard.o")
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-DKID_GUARD", "-c", "-o", gobj,
           os.path.join(CSRC, "kid_capi.cu")]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    out = os.path.join(PKG, "libkernid_cuda_guard.so")
    objs = [gobj] + [os.path.join(objdir, f[:-3] + ".o") for f in CU_SRCS if f != "kid_capi.cu"]
    subprocess.run([NVCC, *ARCH, "-shared", "-o", out] + objs, check=True)
    return out


def build_host(force=False, verbose=False):
    if not os.path.isdir(HOST):
        return None
    deps = [os.path.join(HOST, f) for f in os.listdir(HOST)] + [os.path.join(ROOT, "include", f)
                                                                for f in os.listdir(os.path.join(ROOT, "include"))]
    if not force and not _stale(HOST_SO, deps):
        return HOST_SO
    cmd = ["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-ffp-contract=off", "-Wall",
           "-I", os.path.join(ROOT, "include"), "-o", HOST_SO] + [os.path.join(HOST, f) for f in HOST_SRCS] + \
          ["-I", "/usr/local/cuda/include", "-L", PKG, "-lkernid_cuda", "-Wl,-rpath,$ORIGIN",
           "-L/usr/lib/x86_64-linux-gnu", "-l:libnccl.so.2", "-ldl", "-lpthread"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return HOST_SO


def build_all(force=False, verbose=False):
    cuda_rebuilt = _stale(CUDA_SO, [os.path.join(CSRC, f) for f in os.listdir(CSRC)])
    build_cuda(force, verbose)
    build_host(force or cuda_rebuilt, verbose)


if __name__ == "__main__":
    if "--guard" in sys.argv:
        print(build_guard(verbose=True))
    else:
        build_all(force="--force" in sys.argv, verbose=True)
