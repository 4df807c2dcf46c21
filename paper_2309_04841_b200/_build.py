"""Build libfqaoa.so (sm_100a) in-tree with nvcc.

``python -m paper_2309_04841_b200._build`` or ``__graft_entry__.build()``.
The library lands next to this file so it travels with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libfqaoa.so")
SOURCES = ["ops.cu", "evolve.cu", "pass_rx_u16_light.cu", "pass_rx_u16_heavy.cu", "pass_rx_f64_light.cu",
           "pass_rx_f64_heavy.cu", "pass_su2.cu", "pass_su2_c64.cu", "pass_c64_u16.cu", "pass_c64_f64.cu", "pass_global_u16.cu",
           "pass_global_f64.cu", "pass_global_c64.cu", "xy.cu", "global.cu",
           "wht.cu", "sweep.cu", "sweep_c128_k3.cu", "sweep_c128_k4.cu", "sweep_c64_k3.cu", "sweep_c64_k4.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def host_compiler() -> list[str]:
    # the image's default `gcc` wrapper lacks some spec files; prefer the system one
    for cand in ("/usr/bin/g++",):
        if os.path.exists(cand):
            return ["-ccbin", cand]
    return []


def _headers() -> list[str]:
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + \
        [os.path.join(INCLUDE, "fqaoa.h"), __file__]


STAMP = LIB + ".stamp"


def _digest() -> str:
    """Content hash of every build input (robust to mtime changes when the
    tree is copied, e.g. to the GPU box)."""
    import hashlib

    h = hashlib.sha256()
    for path in sorted([os.path.join(CSRC, f) for f in SOURCES] + _headers()):
        with open(path, "rb") as f:
            h.update(os.path.basename(path).encode() + b"\0" + f.read())
    return h.hexdigest()


def _stale() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as f:
        return f.read().strip() != _digest()


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    """Compile every translation unit (in parallel; an object is rebuilt when
    its source or any header is newer) and link libfqaoa.so."""
    if not force and not _stale():
        return LIB
    tmpdir = os.path.join(HERE, "build")
    os.makedirs(tmpdir, exist_ok=True)
    common = [nvcc(), *host_compiler(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-I", INCLUDE, "-I", CSRC, "--expt-relaxed-constexpr"]
    if verbose:
        common += ["-Xptxas", "-v"]
    hdr_t = max(os.path.getmtime(h) for h in _headers())
    objs, procs = [], []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(tmpdir, src.replace(".cu", ".o"))
        objs.append(obj)
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(hdr_t, os.path.getmtime(path)):
            continue
        procs.append((src, [*common, "-c", path, "-o", obj]))
    jobs = jobs or max(1, min(len(procs), os.cpu_count() or 1))
    running: list = []
    failed = []

    def reap(block: bool) -> None:
        for item in list(running):
            src, p = item
            if block or p.poll() is not None:
                out, err = p.communicate()
                if p.returncode != 0 or verbose:
                    sys.stderr.write(out + err)
                if p.returncode != 0:
                    failed.append(src)
                running.remove(item)

    for src, cmd in procs:
        while len(running) >= jobs:
            reap(False)
            if len(running) >= jobs:
                running[0][1].wait()
        running.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    reap(True)
    if failed:
        raise RuntimeError(f"nvcc failed on {', '.join(failed)}")
    tmp_lib = LIB + ".tmp"
    cmd = [nvcc(), *host_compiler(), *ARCH, "-shared", "-o", tmp_lib, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp_lib, LIB)
    with open(STAMP, "w") as f:
        f.write(_digest() + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
