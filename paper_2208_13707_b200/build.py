"""Build libmpix.so in-tree for sm_100a (nvcc, no JIT cache).

The shared library holds the C++ host runtime (csrc/mpix_runtime.cpp), the
sm_100a kernels (csrc/mpix_kernels.cu) and the test/bench helper kernels
(csrc/mpix_testing.cu). It travels with the repo snapshot to the GPU box.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmpix.so")
SOURCES = ["mpix_runtime.cpp", "mpix_p2p.cpp", "mpix_coll.cpp", "mpix_heap.cpp", "mpix_kernels.cu",
           "mpix_testing.cu", "mpix_drivers.cpp"]
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps += [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not needs_build():
        return LIB
    objs = []
    odir = os.path.join(HERE, "_obj")
    os.makedirs(odir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
              "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
    cmds = []
    for src in SOURCES:
        obj = os.path.join(odir, src + ".o")
        cmd = [nvcc(), ARCH, *common, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu") and verbose:
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        cmds.append(cmd)
        objs.append(obj)
    # translation units compile in parallel (the kernels TU dominates)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 4)) as ex:
        for r in list(ex.map(lambda c: subprocess.run(c), cmds)):
            if r.returncode != 0:
                raise subprocess.CalledProcessError(r.returncode, r.args)
    tmp = LIB + ".tmp"
    cmd = [nvcc(), ARCH, "-shared", "-o", tmp, *objs, "-lpthread",
           "-Xlinker", "--version-script=" + os.path.join(CSRC, "exports.map")]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


def build_tsan(verbose=False):
    """libmpix_tsan.so: the same sources with the host code built under
    ThreadSanitizer (-fsanitize=thread), for tools/sanitize.sh (load it with
    MPIX_LIB_PATH and LD_PRELOAD=libtsan.so). Not used by the product."""
    out = os.path.join(HERE, "libmpix_tsan.so")
    odir = os.path.join(HERE, "_obj_tsan")
    os.makedirs(odir, exist_ok=True)
    common = ["-O1", "-g", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fsanitize=thread",
              "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
    objs, cmds = [], []
    for src in SOURCES:
        obj = os.path.join(odir, src + ".o")
        cmds.append([nvcc(), ARCH, *common, "-c", os.path.join(CSRC, src), "-o", obj])
        objs.append(obj)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 4)) as ex:
        for r in list(ex.map(lambda c: subprocess.run(c), cmds)):
            if r.returncode != 0:
                raise subprocess.CalledProcessError(r.returncode, r.args)
    subprocess.run([nvcc(), ARCH, "-shared", "-o", out, *objs, "-lpthread", "-Xcompiler", "-fsanitize=thread",
                    "-Xlinker", "--version-script=" + os.path.join(CSRC, "exports.map")], check=True)
    return out


if __name__ == "__main__":
    if "--tsan" in sys.argv:
        print(build_tsan())
        sys.exit(0)
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
