"""Build the native library in-tree: libldurepart_b200.so (sm_100a only).

    python -m paper_2510_08536_b200.build        # or __graft_entry__.build()

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libldurepart_b200.so")
# separately compiled translation units (built in parallel, then linked)
SOURCES = ["plan.cpp", "device.cu", "scatter.cu", "solve_cg.cu", "solve_bicgstab.cu", "solve_pcg1.cu", "solve_pipecg.cu", "solve_pipecg_t.cu"]
HEADERS = ["lrb_internal.h", "kernels.cuh", "stream.cuh", "launch.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMPILE_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xptxas", "-v", "--expt-relaxed-constexpr",
                 "-Xcompiler", "-fPIC,-O3,-pthread,-Wall,-Wno-unused-function"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build ldurepart_b200")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "ldurepart_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, extra=()) -> str:
    """Compile the library; ``out``/``extra`` build tuning variants (e.g. -DLRB_MINB=3).
    Each translation unit is compiled by its own nvcc process (in parallel),
    then the objects are linked into one shared library."""
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    tag = os.path.basename(lib).replace(".so", "")
    objdir = os.path.join(HERE, "build", tag)
    os.makedirs(objdir, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [nvcc(), *ARCH, *COMPILE_FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                                 text=True)))
    logs, objs, failed = [], [], False
    for src, obj, p in procs:
        out_s, err_s = p.communicate()
        logs.append(f"==== {src}\n{out_s}{err_s}")
        objs.append(obj)
        if p.returncode != 0:
            failed = True
            sys.stderr.write(out_s + err_s)
    if failed:
        raise RuntimeError("ldurepart_b200 native build failed")
    res = subprocess.run([nvcc(), *ARCH, "-shared", "-Xcompiler", "-pthread", *objs, "-o", lib + ".tmp"],
                         capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("ldurepart_b200 native link failed")
    if out is None:
        with open(os.path.join(HERE, "csrc", "ptxas.log"), "w") as fh:
            fh.write("\n".join(logs))
    if verbose:
        sys.stderr.write("\n".join(logs))
    os.replace(lib + ".tmp", lib)
    return lib


PROF_LIB = os.path.join(HERE, "libldurepart_b200_prof.so")


def build_profiling(force: bool = False) -> str:
    """Diagnostics variant with the streaming solvers' wait/issue counters
    compiled in (-DLRB_PROF=1); select it with LRB_LIB=<path> (tools/)."""
    if not force and os.path.exists(PROF_LIB) and os.path.getmtime(PROF_LIB) >= os.path.getmtime(LIB) \
            and not _stale():
        return PROF_LIB
    return build(force=True, out=PROF_LIB, extra=["-DLRB_PROF=1"])


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    print(build_profiling(force="--force" in sys.argv))
