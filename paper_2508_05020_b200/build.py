"""Build the in-tree C-ABI library ``libamr.so`` (sm_100a) with nvcc.

    python -m paper_2508_05020_b200.build [--force] [--verbose-ptxas]

Sources: csrc/*.cu, csrc/*.cpp.  Output: paper_2508_05020_b200/libamr.so (git-ignored,
travels to the GPU box with the repo snapshot).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libamr.so")
BUILD = os.path.join(HERE, "..", "build", "amr")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_include():
    try:
        import nvidia.nccl  # noqa: F401
        base = os.path.dirname(sys.modules["nvidia.nccl"].__file__ or list(sys.modules["nvidia.nccl"].__path__)[0])
    except Exception:
        base = None
    cands = []
    if base:
        cands.append(os.path.join(base, "include"))
    cands += glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "nccl", "include"))
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    return None


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(HERE, "..", "include", "amr.h")])


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose_ptxas: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    inc = ["-I", CSRC, "-I", os.path.join(HERE, "..", "include")]
    nccl_inc = _nccl_include()
    if nccl_inc:
        inc += ["-I", nccl_inc, "-DAMR_HAVE_NCCL_H=1"]
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall"] + ARCH + inc
    common += os.environ.get("AMR_NVCC_FLAGS", "").split()   # e.g. -DAMR_PHASE_PROF (kernel phase timing)
    stamp = os.path.join(BUILD, "flags.txt")   # objects built with other flags are stale
    prev = open(stamp).read() if os.path.exists(stamp) else None
    if prev != " ".join(common):
        force = True
    objs, jobs = [], []
    hdrs = headers()
    for src in sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            extra = ["-Xptxas", "-v"] if (verbose_ptxas and src.endswith(".cu")) else []
            jobs.append([NVCC, "-c", src, "-o", obj] + common + extra)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    failed = []
    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for cmd, r in ex.map(run, jobs):
            if r.returncode != 0:
                failed.append((cmd, r))
            elif verbose_ptxas and r.stderr:
                sys.stderr.write(r.stderr)
    if failed:
        for cmd, r in failed:
            sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError("nvcc failed")
    if force or jobs or _stale(OUT, objs):
        cmd = [NVCC, "-shared", "-o", OUT + ".tmp"] + objs + ARCH + ["-cudart=static", "-ldl", "-lpthread"]
        subprocess.check_call(cmd)
        os.replace(OUT + ".tmp", OUT)
    with open(stamp, "w") as f:
        f.write(" ".join(common))
    return OUT


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose-ptxas", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose_ptxas=a.verbose_ptxas))
