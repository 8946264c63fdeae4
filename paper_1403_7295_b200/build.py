"""Build recipe for libpaes_cuda.so (in-tree, sm_100a only).

    python -m paper_1403_7295_b200.build          # or __graft_entry__.build()

nvcc cross-compiles for sm_100a without a GPU; the .so lands in
paper_1403_7295_b200/lib/ so it travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libpaes_cuda.so")
SOURCES = ["aes_kernels.cu", "runtime.cu", "abi_core.cu", "abi_batch.cu", "abi_file.cu", "host_rules.cpp", "host_copy.cpp"]
HEADERS = ["aes_kernels.cuh", "aes_tables.hpp", "host_rules.hpp", "host_copy.hpp", "launch.hpp", "runtime.hpp", "sbox_bitsliced.inc",
           "gpu_worker.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# system g++: links libstdc++ dynamically, like the torch/numpy in the same process
CCBIN = ["-ccbin", "/usr/bin/g++"] if os.path.exists("/usr/bin/g++") else []
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v",
         f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "paes_cuda.h"),
                                                                 os.path.abspath(__file__)]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out_lib: str | None = None,
          host_flags=()) -> str:
    """Compile + link.  `defines` (e.g. ["PAES_NB=4"]), `host_flags` (e.g.
    ["-fsanitize=thread"], host compiler + link) and `out_lib` are for variants
    (scripts/tune_variants.py, scripts/tsan_stress.sh); the product uses the
    defaults."""
    lib = out_lib or LIB
    if not force and out_lib is None and not _stale():
        _build_aux(missing_only=True)
        return LIB
    lib_dir = os.path.dirname(lib)
    os.makedirs(lib_dir, exist_ok=True)
    dflags = ["-D" + d for d in defines]
    hflags = ["-Xcompiler", ",".join(host_flags)] if host_flags else []
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):
        obj = os.path.join(lib_dir, src + ".o")
        cmd = [NVCC] + CCBIN + ARCH + FLAGS + dflags + hflags + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s%s" % (src, r.stdout, r.stderr))
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib + ".tmp"
    cmd = [NVCC] + CCBIN + ARCH + hflags + ["-shared", "-o", tmp] + objs + ["-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n%s%s" % (r.stdout, r.stderr))
    os.replace(tmp, lib)
    for o in objs:
        os.unlink(o)
    if out_lib is None:
        _build_aux()
    return lib


def _build_aux(missing_only: bool = False) -> None:
    """The executables and libraries built next to libpaes_cuda.so."""
    for path, fn in ((WORKER, build_worker), (BITSLICED_AB, build_bitsliced_ab), (AES_ABI, build_aes_abi)):
        if not missing_only or not os.path.exists(path):
            fn()


BITSLICED_AB = os.path.join(LIB_DIR, "libpaes_bitsliced_ab.so")


def build_bitsliced_ab() -> str:
    """The bitsliced (LOP3) encrypt kernel of the north_star T-table vs
    bitsliced A/B, in a library of its own so the product .so carries only the
    shipped kernels (csrc/aes_bitsliced.cu + the host key rules)."""
    tmp = BITSLICED_AB + ".tmp"
    cmd = [NVCC] + CCBIN + ARCH + FLAGS + ["-shared", "-o", tmp, os.path.join(CSRC, "aes_bitsliced.cu"),
                                           os.path.join(CSRC, "host_rules.cpp")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("bitsliced A/B build failed:\n%s%s" % (r.stdout, r.stderr))
    os.replace(tmp, BITSLICED_AB)
    return BITSLICED_AB


WORKER = os.path.join(LIB_DIR, "paes_gpu_worker")


def build_worker() -> str:
    """The reference-protocol GPU worker executable (csrc/gpu_worker.cpp)."""
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [cxx, "-std=c++17", "-O2", "-Wall", "-Wextra", f"-I{os.path.join(ROOT, 'include')}",
           os.path.join(CSRC, "gpu_worker.cpp"), "-o", WORKER + ".tmp", f"-L{LIB_DIR}", "-lpaes_cuda",
           "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("worker build failed:\n%s%s" % (r.stdout, r.stderr))
    os.replace(WORKER + ".tmp", WORKER)
    return WORKER


AES_ABI = os.path.join(LIB_DIR, "libpaes_aes_b200.so")


def build_aes_abi() -> str:
    """libpaes_aes_b200.so: the reference's aes.cpp entry points (aes.hpp
    mangled C++ symbols) backed by libpaes_cuda.so -- the link-level drop-in
    (csrc/aes_cxx_abi.cpp)."""
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [cxx, "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", f"-I{os.path.join(ROOT, 'include')}",
           os.path.join(CSRC, "aes_cxx_abi.cpp"), "-o", AES_ABI + ".tmp", f"-L{LIB_DIR}", "-lpaes_cuda",
           "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("aes ABI library build failed:\n%s%s" % (r.stdout, r.stderr))
    os.replace(AES_ABI + ".tmp", AES_ABI)
    return AES_ABI


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
