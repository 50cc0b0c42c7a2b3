"""Build libhh.so (the C-ABI CUDA library) in-tree for sm_100a with nvcc."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhh.so")
SOURCES = ["hh_api.cu", "fine2d.cu", "fine3d.cu", "coarse_nd.cu", "krylov.cu", "comm.cu", "lfa.cu", "peak.cu", "fd.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-cudart", "shared", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-ldl"]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "hh.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    """Compile every source to an object in parallel (nvcc -c), then link."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f not in ("-shared", "-ldl")]

    def comp(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        r = subprocess.run([NVCC] + cflags + ["-c", "-o", obj, os.path.join(CSRC, src)],
                           capture_output=True, text=True)
        return src, obj, r

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        res = list(ex.map(comp, SOURCES))
    log = "".join(r.stdout + r.stderr for _, _, r in res)
    bad = [src for src, _, r in res if r.returncode]
    if verbose or bad:
        sys.stderr.write(log)
    if bad:
        raise RuntimeError("nvcc failed building libhh.so: " + ", ".join(bad))
    r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "shared",
                        "-o", LIB] + [o for _, o, _ in res] + ["-ldl"], capture_output=True, text=True)
    if verbose or r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode:
        raise RuntimeError("nvcc failed linking libhh.so")
    with open(os.path.join(HERE, "ptxas.log"), "w") as f:
        f.write(log)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
