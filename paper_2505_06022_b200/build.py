"""Build ``libcq.so`` in-tree for sm_100a with nvcc (no JIT cache, so the
built library travels to the GPU box with the repository snapshot).

    python -m paper_2505_06022_b200.build [--force]
"""

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libcq.so")
SOURCES = ["cq_runtime.cu", "cq_kernels.cu", "cq_sgemm.cu", "cq_tf32.cu", "cq_nvml.cu", "cq_plan.cpp",
           "cq_jit.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _nccl_rpath():
    """Directories searched for libnccl.so.2 at run time.  The NCCL that
    PyTorch ships (nvidia-nccl wheel) comes first, so libcq and torch share
    one NCCL whichever of them is loaded first (two different libnccl.so.2
    in one process break the later one); the system copy is the fallback."""
    import importlib.util
    dirs = []
    spec = importlib.util.find_spec("nvidia.nccl")
    for base in (spec.submodule_search_locations or []) if spec else []:
        lib = os.path.join(base, "lib")
        if os.path.exists(os.path.join(lib, "libnccl.so.2")):
            dirs.append(lib)
    return dirs + ["/usr/lib/x86_64-linux-gnu", "/usr/local/cuda/lib64"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers():
    hs = [os.path.join(ROOT, "include", "cq.h")]
    hs += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs


def build(force=False, verbose=False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    heads = _headers()
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        if force or _stale(o, [s] + heads):
            jobs.append((s, o))

    def compile_one(job):
        s, o = job
        cmd = [NVCC, *ARCH, *FLAGS, "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(OBJ, os.path.basename(s) + ".log")
        with open(log, "w") as fh:
            fh.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{r.stderr[-6000:]}")
        return s

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for s in ex.map(compile_one, jobs):
            if verbose:
                print("compiled", os.path.relpath(s, ROOT))
    objs = [os.path.join(OBJ, s + ".o") for s in SOURCES]
    if force or jobs or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lnccl", "-lnvrtc", "-ldl",
               "-Xlinker", "-rpath," + ":".join(_nccl_rpath())]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
        if verbose:
            print("linked", os.path.relpath(LIB, ROOT))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
