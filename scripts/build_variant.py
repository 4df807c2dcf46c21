"""Development A/B builds: compile libfqaoa.so's sources with extra nvcc
defines into paper_2309_04841_b200/variants/<name>/libfqaoa.so (objects under
build/variants/, which stays on this machine; the .so travels with gpurun), reusing
the main build's objects for units that do not include pass.cuh.  Select one at
run time with FQ_LIB_VARIANT=<name> (timing experiments only).

    python scripts/build_variant.py nopair -DFQ_PAIR_RX=0
"""

import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_04841_b200 import _build  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    _build.build()
    out = os.path.join(_build.HERE, "build", "variants", name)
    lib_dir = os.path.join(_build.HERE, "variants", name)
    os.makedirs(out, exist_ok=True)
    os.makedirs(lib_dir, exist_ok=True)
    common = [_build.nvcc(), *_build.host_compiler(), *_build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler",
              "-fPIC", "-I", _build.INCLUDE, "-I", _build.CSRC, "--expt-relaxed-constexpr", *defs]
    objs, procs = [], []
    for src in _build.SOURCES:
        text = open(os.path.join(_build.CSRC, src)).read()
        if "pass.cuh" in text or "tmap.cuh" in text:
            obj = os.path.join(out, src.replace(".cu", ".o"))
            procs.append(subprocess.Popen([*common, "-c", os.path.join(_build.CSRC, src), "-o", obj]))
        else:
            obj = os.path.join(_build.HERE, "build", src.replace(".cu", ".o"))
        objs.append(obj)
    if any(p.wait() for p in procs):
        raise SystemExit("nvcc failed")
    subprocess.check_call([_build.nvcc(), *_build.host_compiler(), *_build.ARCH, "-shared", "-o",
                           os.path.join(lib_dir, "libfqaoa.so"), *objs])
    print(os.path.join(lib_dir, "libfqaoa.so"))


if __name__ == "__main__":
    main()
