"""Build libmpx.so in-tree with nvcc for sm_100a.

    python paper_2402_12274_b200/build.py [--force] [-v]

One shared library from csrc/*.cu + csrc/*.cpp, static cudart, -lineinfo so
ncu's source page maps to the kernels.  The .so is git-ignored but travels to
the GPU box with the gpurun snapshot.
"""

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(os.path.dirname(HERE), "include")
SO = os.environ.get("MPX_SO_OUT") or os.path.join(HERE, "libmpx.so")   # MPX_SO_OUT: A/B builds
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-Wall",
         "--expt-relaxed-constexpr", "-I", CSRC, "-I", INC] + \
    os.environ.get("MPX_NVCC_FLAGS", "").split()   # experiments only (e.g. -DMPX_PERM_BPS2=3)


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) +
                  glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h*")) + \
        glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INC, "*.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False):
    if not force and not _stale():
        return SO
    objdir = os.path.join(HERE, "_obj") if SO.endswith(os.path.join(HERE, "libmpx.so")) else SO + ".obj"
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC] + ARCH + FLAGS + ["-x", "cu" if src.endswith(".cu") else "c++",
                                       "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                            stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = False
    for cmd, p in procs:
        out = p.communicate()[0].decode(errors="replace")
        if p.returncode != 0:
            failed = True
            sys.stderr.write("FAILED: %s\n%s\n" % (" ".join(cmd), out))
        elif verbose and out.strip():
            sys.stderr.write(out)
    if failed:
        raise RuntimeError("libmpx build failed")
    link = [NVCC] + ARCH + ["-shared", "-o", SO + ".tmp"] + objs + \
        ["-ldl", "-lpthread", "-lrt"]
    subprocess.check_call(link)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
