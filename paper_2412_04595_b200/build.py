"""Build libsog.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "libsog.so")
SOURCES = ["sog_api.cu", "mid.cu", "long.cu", "dft.cu", "fft.cu", "near.cu", "scan.cu", "plan.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = (["-DSOG_ASSERTS"] if os.environ.get("SOG_ASSERTS") else []) + ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _obj_stale(src: str, obj: str) -> bool:
    """An object is stale when it, or its nvcc -MD dependency file, is older than any dependency."""
    dep = obj + ".d"
    if not (os.path.exists(obj) and os.path.exists(dep)):
        return True
    t = os.path.getmtime(obj)
    with open(dep) as f:
        text = f.read().replace("\\\n", " ")
    files = [w for w in text.split(":", 1)[-1].split() if w]
    files.append(os.path.join(CSRC, src))
    return any(not os.path.exists(d) or os.path.getmtime(d) > t for d in files)


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for root in (CSRC, os.path.join(os.path.dirname(HERE), "include")):
        for f in os.listdir(root):
            if os.path.getmtime(os.path.join(root, f)) > t:
                return True
    return False


def build(force: bool = False, verbose: bool = False) -> str:
    stamp = os.path.join(HERE, "lib", "obj", "flags.txt")
    flags = " ".join(FLAGS)
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        force = True               # compiler flags changed (e.g. SOG_ASSERTS): rebuild everything
    if not force and not _stale():
        return LIB
    os.makedirs(os.path.join(HERE, "lib", "obj"), exist_ok=True)
    with open(stamp, "w") as f:
        f.write(flags)
    objs, procs = [], []
    for src in SOURCES:            # one nvcc per stale translation unit, in parallel
        obj = os.path.join(HERE, "lib", "obj", src + ".o")
        objs.append(obj)
        if not force and not _obj_stale(src, obj):
            continue
        cmd = [NVCC, *FLAGS, "-MD", "-MF", obj + ".d", "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd), cmd))
    for pr, cmd in procs:
        if pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, cmd)
    link = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", LIB + ".tmp",
            "-L/usr/local/cuda/lib64", "-lcufft", "-lquadmath", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    subprocess.run(link, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
