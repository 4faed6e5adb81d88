"""Build the in-tree CUDA libraries with nvcc for sm_100a (no JIT, no torch extension machinery).

  libvnm.so                    the product: C ABI of include/vnm.h (api.cpp + the kernels in csrc/)
  tests/probes/libvnm_probe.so test-only hardware probes / microbenchmarks (tests/probes/probes*.cu); the
                               product never loads it
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2",
         "-Xptxas", "-warn-spills"]

PROBES = os.path.join(HERE, "..", "tests", "probes")
# output path -> (source directory, sources)
LIBS = {
    os.path.join(HERE, "libvnm.so"): (CSRC, ["api.cpp", "prune.cu", "prune2.cu", "spmm.cu", "pack_tc.cu",
                                           "spmm_tc.cu", "spmm_tc2.cu", "spmm_tc3.cu", "spmm_smallt.cu", "ria.cu", "permute.cu", "permute_out.cu"]),
    os.path.join(PROBES, "libvnm_probe.so"): (PROBES, ["probes.cu", "probes2.cu", "probes3.cu", "probes4.cu"]),
}


def _stale(out: str, srcs: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(HERE, "..", "include", "vnm.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, ablations: bool = False) -> None:
    """Each source is compiled to an object in build/ (in parallel, only when stale), then linked.
    ablations=True builds libvnm_abl.so instead (-DVNM_ABLATIONS: the VNM_ABL timing switches; results invalid;
    experiments only, loaded when VNM_LIB points at it)."""
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build_abl" if ablations else "build")
    os.makedirs(objdir, exist_ok=True)
    libs = {os.path.join(HERE, "libvnm_abl.so"): LIBS[os.path.join(HERE, "libvnm.so")]} if ablations else LIBS
    extra = ["-DVNM_ABLATIONS"] if ablations else []
    for out, (srcdir, files) in libs.items():
        srcs = [os.path.join(srcdir, f) for f in files]
        if not force and not _stale(out, srcs):
            continue
        objs = [os.path.join(objdir, f + ".o") for f in files]

        def compile_one(i):
            if not force and not _stale(objs[i], [srcs[i]]):
                return
            tmp = objs[i] + f".tmp{os.getpid()}"
            cmd = [NVCC, *ARCH, *FLAGS, *extra, "-I", CSRC, "-c", "-o", tmp, srcs[i]]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.check_call(cmd)
            os.replace(tmp, objs[i])

        with ThreadPoolExecutor(max_workers=min(8, len(files))) as ex:
            list(ex.map(compile_one, range(len(files))))
        tmp = out + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        os.replace(tmp, out)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ablations="--ablations" in sys.argv)
