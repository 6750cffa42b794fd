"""Build the sm_100a shared library in-tree (nvcc -shared), no JIT cache.

    python -m paper_2605_16082_b200.build
produces paper_2605_16082_b200/libprismdg_b200.so (git-ignored; travels to the GPU box).
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libprismdg_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O3",
         "-I" + os.path.join(ROOT, "include")]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "prismdg_b200.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(verbose=False, force=False, extra=(), out=None):
    """out: alternative library path (A/B builds with extra -D flags); default the in-tree library."""
    if out is None and not force and not needs_build():
        return LIB
    objdir = os.path.join(ROOT, "build", "obj" if out is None else "obj_" + os.path.basename(out))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = ["nvcc", *ARCH, *FLAGS, *extra, "-dc" if False else "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        log = p.communicate()[0].decode()
        if p.returncode != 0 or verbose:
            sys.stderr.write(log)
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    cmd = ["nvcc", *ARCH, "-shared", "-o", out or LIB, *objs, "-lcudart", "-ldl"]
    subprocess.check_call(cmd)
    return out or LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force=True)
    print(LIB)
