"""Build recipe for the native library (sm_100a only).

    python -m paper_2003_11076_b200.build          # builds lib/libseethrough_b200.so

The library is built in-tree so it travels with the repository snapshot to
the GPU box; it is git-ignored.
"""

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libseethrough_b200.so")
SOURCES = ["st_api.cu", "st_em.cu", "st_features.cu", "st_frame.cu", "st_harvest.cu",
           "st_host.cu", "st_mean.cu", "st_mu.cu", "st_prior.cu", "st_refocus.cu",
           "st_render.cu"]
HEADERS = ["st_common.cuh", "st_em.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _inputs():
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "seethrough_b200.h"))
    return files


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _inputs())


def build(force=False, verbose=False, jobs=None, defines=(), out=None):
    """Compile every .cu for sm_100a and link one shared library.

    defines / out: an experiment variant (-D flags) linked to another path
    (load it with ST_LIB_PATH=<out>); the default library is untouched."""
    lib = out or LIB
    if not force and not defines and out is None and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj" if out is None else "obj_" + os.path.basename(out))
    os.makedirs(objdir, exist_ok=True)
    common = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--extended-lambda",
                     "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
                     "-Xptxas", "-v"] + ["-D" + d for d in defines]
    procs = []
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [NVCC] + common + ["-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    logs = []
    for src, pr in procs:
        out, _ = pr.communicate()
        logs.append(out.decode(errors="replace"))
        if pr.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{logs[-1]}")
    tmp = lib + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-cudart", "static", "-ldl",
                                                          "-Xcompiler", "-pthread"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stdout.decode(errors="replace"))
    os.replace(tmp, lib)
    with open(lib + ".ptxas.log", "w") as fh:  # ptxas -v: registers / spills per kernel
        fh.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
