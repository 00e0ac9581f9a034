"""Build libmnl.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib", "libmnl.so")
HOST_OUT = os.path.join(HERE, "lib", "libnrhost.so")   # the same NR driver over host callbacks (CPU tests)
SOURCES = ["mnl_api.cu", "k_eval.cu", "k_eval_w.cu", "k_eval_w1.cu", "k_eval_w2.cu", "k_eval_x.cu", "k_hess.cu", "k_chol.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-Xptxas", "-v",
         *os.environ.get("MNL_NVCC_EXTRA", "").split()]


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, "internal.h"),
                                                       os.path.join(CSRC, "eval_common.h"),
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
    # one nvcc per translation unit, in parallel, then one link (no cross-unit device code)
    objdir = os.path.join(HERE, "lib", "obj")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"]
    jobs, text = [], ""
    hdrs = [os.path.join(CSRC, "internal.h"), os.path.join(CSRC, "eval_common.h"), os.path.join(CSRC, "k_eval_w.cu"), os.path.join(CSRC, "nr_driver.h"),
            os.path.join(HERE, "..", "include", "mnl.h")]
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *cflags, "-c", "-o", obj, os.path.join(CSRC, src)]
        if not force and os.path.exists(obj) and all(
                os.path.getmtime(obj) > os.path.getmtime(p) for p in [os.path.join(CSRC, src), *hdrs]):
            jobs.append((cmd, obj, None))  # up to date
            continue
        jobs.append((cmd, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    failed = False
    for cmd, _, pr in jobs:
        if pr is None:
            continue
        out, err = pr.communicate()
        text += " ".join(cmd) + "\n" + out + err
        failed |= pr.returncode != 0
    log = os.path.join(HERE, "lib", "build.log")
    if not failed:
        tmp = OUT + f".tmp{os.getpid()}"
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", tmp,
               *[obj for _, obj, _ in jobs]]
        r = subprocess.run(cmd, capture_output=True, text=True)
        text += " ".join(cmd) + "\n" + r.stdout + r.stderr
        failed = r.returncode != 0
        if not failed:
            os.replace(tmp, OUT)
    with open(log, "w") as fh:
        fh.write(text)
    if failed:
        sys.stderr.write(text[-20000:])
        raise RuntimeError(f"nvcc failed; see {log}")
    if verbose:
        sys.stderr.write(text)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
