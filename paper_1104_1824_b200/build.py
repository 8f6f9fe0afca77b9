"""Build the in-tree CUDA libraries for sm_100a (no JIT cache, no CPU path).

* ``libsnp.so``     — the engine: kernels + C ABI of include/snp.h
* ``libsnpgen.so``  — device-side level-0 input generator (workloads only)
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_SNP = os.path.join(HERE, "libsnp.so")
LIB_GEN = os.path.join(HERE, "libsnpgen.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]

SNP_SOURCES = ["snp_engine.cu", "snp_kernels.cu", "snp_comm.cu"]
SNP_DEPS = SNP_SOURCES + ["snp_device.cuh", "snp_internal.h", "snp_tc.cuh", "snp_comm.h", "../../include/snp.h"]
LIBS = ["-ldl"]  # libnccl.so.2 is opened at run time (snp_comm.cu)


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(os.path.join(CSRC, d)) > t for d in deps)


def _nvcc(out: str, sources, extra=()):
    """compile each source to an object in parallel (-dc free: no device
    linking across files), then link the shared library"""
    from concurrent.futures import ThreadPoolExecutor
    tmp = out + f".tmp{os.getpid()}"
    objs = [f"{tmp}.{i}.o" for i in range(len(sources))]
    comp = [x for x in FLAGS if x != "-shared"]

    def one(i):
        subprocess.check_call([NVCC, *ARCH, *comp, *extra, "-c", "-o", objs[i], os.path.join(CSRC, sources[i])])

    try:
        with ThreadPoolExecutor(len(sources)) as ex:
            list(ex.map(one, range(len(sources))))
        subprocess.check_call([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs, *LIBS])
        os.replace(tmp, out)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.unlink(o)


def build(force: bool = False, verbose: bool = False) -> None:
    if force or _stale(LIB_SNP, SNP_DEPS):
        if verbose:
            print("[build] nvcc libsnp.so (sm_100a)")
        _nvcc(LIB_SNP, SNP_SOURCES)
    if force or _stale(LIB_GEN, ["workload_gen.cu"]):
        if verbose:
            print("[build] nvcc libsnpgen.so (sm_100a)")
        _nvcc(LIB_GEN, ["workload_gen.cu"])


def build_variant(out: str, defines) -> None:
    """Tuning aid: build libsnp.so with extra -D defines to another path."""
    _nvcc(out, SNP_SOURCES, [f"-D{d}" for d in defines])


if __name__ == "__main__":
    build(force=True, verbose=True)
