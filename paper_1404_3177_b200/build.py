"""Build libmnl.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib", "libmnl.so")
HOST_OUT = os.path.join(HERE, "lib", "libnrhost.so")   # the same NR driver over host callbacks (CPU tests)
SOURCES = ["mnl_api.cu", "k_eval.cu", "k_hess.cu", "k_chol.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-Xptxas", "-v"]


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, "internal.h"),
                                                       os.path.join(CSRC, "nr_driver.h"),
                                                       os.path.join(HERE, "..", "include", "mnl.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build_host(force: bool = False) -> str:
    """g++ -> lib/libnrhost.so (no CUDA): nr_driver.h over host callbacks."""
    src = [os.path.join(CSRC, "nr_host.cpp"), os.path.join(CSRC, "nr_driver.h")]
    if force or not os.path.exists(HOST_OUT) or any(os.path.getmtime(p) > os.path.getmtime(HOST_OUT) for p in src):
        os.makedirs(os.path.dirname(HOST_OUT), exist_ok=True)
        tmp = HOST_OUT + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-o", tmp, src[0]])
        os.replace(tmp, HOST_OUT)
    return HOST_OUT


def build(force: bool = False, verbose: bool = False) -> str:
    build_host(force)
    if not force and not stale():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = [NVCC, *FLAGS, "-o", OUT, *[os.path.join(CSRC, s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "lib", "build.log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed ({r.returncode}); see {log}")
    if verbose:
        sys.stderr.write(r.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
