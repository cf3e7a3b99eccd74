"""Build libvpe.so in-tree: nvcc -gencode arch=compute_100a,code=sm_100a for every csrc/*.cu.

Objects are compiled in parallel and linked with the static CUDA runtime; the resulting
``paper_2508_11584_b200/libvpe.so`` travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# diagnostics variants build side by side: VPE_BUILD_TAG=trace -> libvpe_trace.so (loaded with
# VPE_LIB=libvpe_trace.so); the product library is always libvpe.so
_TAG = os.environ.get("VPE_BUILD_TAG", "")
OUT = os.path.join(HERE, f"libvpe_{_TAG}.so" if _TAG else "libvpe.so")
OBJ = os.path.join(HERE, f"build_{_TAG}" if _TAG else "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "--expt-relaxed-constexpr",
         "-I", os.path.join(HERE, "..", "include")]
# diagnostics builds only: VPE_NVCC_EXTRA="-DVPE_TRACE_BUILD" compiles the kernels' timeline probes in
FLAGS += os.environ.get("VPE_NVCC_EXTRA", "").split()


# seg.cu: the fused upsample+argmax must round every mul and add separately (torch's order) and
# ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 unless told not to
EXTRA = {"seg.cu": ["--fmad=false"]}


def _stale(src: str, obj: str) -> bool:
    if not os.path.exists(obj):
        return True
    deps = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(HERE, "..", "include", "vpe.h"), src]
    return max(os.path.getmtime(d) for d in deps) > os.path.getmtime(obj)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s) + ".o")
        if force or _stale(s, o):
            jobs.append((s, o))

    def one(job):
        s, o = job
        cmd = [NVCC, *FLAGS, *EXTRA.get(os.path.basename(s), []), "-c", s, "-o", o]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return s, r

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for s, r in ex.map(one, jobs):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed for {s}")
            if verbose and (r.stdout or r.stderr):
                sys.stderr.write(r.stderr)
    objs = [os.path.join(OBJ, os.path.basename(s) + ".o") for s in srcs]
    if force or jobs or not os.path.exists(OUT):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT, *objs,
               "-cudart", "static", "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link of libvpe.so failed")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
