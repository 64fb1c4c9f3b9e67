"""Build libgdp.so in-tree with nvcc for sm_100a (no JIT cache, so the .so travels with the repo)."""
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libgdp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
         "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "550"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu"))) + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh")))


FLAGS_FILE = SO + ".flags"


def _extra():
    return os.environ.get("GDP_NVCC_EXTRA", "").split()   # experiment macros (e.g. -DCOST5_PROF)


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    # the flags the library was built with are stored next to it: a build with other
    # experiment macros is never reused silently
    try:
        with open(FLAGS_FILE) as f:
            if f.read().split() != _extra():
                return True
    except OSError:
        return True
    t = os.path.getmtime(SO)
    hdr = os.path.join(os.path.dirname(HERE), "include", "gdp.h")
    return any(os.path.getmtime(f) > t for f in sources() + [hdr])


def build(force: bool = False) -> str:
    if force or stale():
        cu = [f for f in sources() if f.endswith(".cu")]
        extra = _extra()
        cmd = [NVCC] + FLAGS + extra + ["-o", SO] + cu
        subprocess.check_call(cmd)
        with open(FLAGS_FILE, "w") as f:
            f.write(" ".join(extra))
    return SO


if __name__ == "__main__":
    print(build(force=True))
